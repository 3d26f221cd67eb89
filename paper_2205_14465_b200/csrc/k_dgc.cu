// DGC / top-k h1 on sm_100a: EF-fused sampled-threshold top-k with index
// compaction (DGC is cited at
// P:828 and evaluated at a 1% rate; EF at P:1427).
//
// Pipeline per bucket (every kernel walks a multi-segment table):
//   1. dgc_sample   one CTA per segment: thr = the j*-th largest key of a hashed
//                   stratified sample of acc = g + r (exact k-th key when the
//                   segment fits the sample).  Only an accelerator: the result
//                   cannot depend on thr (reading R3).
//   2. dgc_stream   ONE pass over g and r (12 B/elem): r := acc; candidates
//                   key(acc) >= thr are compacted per warp-run in index order
//                   (ballot/popc); 2048-bin histogram of candidate keys.
//                   The last CTA of a segment picks the radix bin of the k-th key.
//   3. dgc_stream   (fallback mode) only for segments with < k candidates:
//                   recompact with thr = 0 from r.  Adversarial inputs only.
//   4. dgc_refine   two more radix rounds over the candidates -> exact k-th key T,
//                   #above, #ties to take (ties broken by ascending index).
//   5. dgc_count    per group of runs: #above, #ties; last CTA scans offsets.
//   6. dgc_write    ordered selection -> payload idx[]/val[] sorted by index;
//                   EF: r[idx] := 0.
#include <cmath>

#include "esp_device.cuh"
#include "esp_kernels.h"

namespace esp {

// CTA-wide: given a histogram in global memory, find bin b (scanning from the
// top) with above(b) < need <= above(b) + hist[b].  nbins in {1024, 2048}.
__device__ void select_bin(const uint32_t* hist, int nbins, uint32_t need, uint32_t* out_bin,
                           uint32_t* out_above, uint32_t* sh /* >= 256+16 */) {
  const int per = nbins / kThreads;
  const int t = threadIdx.x;
  uint32_t local[8];
  uint32_t sum = 0;
  for (int i = 0; i < per; ++i) {
    local[i] = __ldcg(hist + t * per + i);
    sum += local[i];
  }
  // suffix sums: thread t gets sum over threads > t
  uint32_t* sh_sum = sh;       // 256
  uint32_t* sh_res = sh + 256; // bin, above
  sh_sum[t] = sum;
  __syncthreads();
  uint32_t v = sh_sum[kThreads - 1 - t];
  __syncthreads();
  uint32_t tot;
  uint32_t excl = block_excl_scan(v, &tot, sh + 258);
  // excl over reversed order = sum of threads > (255 - t)
  sh_sum[kThreads - 1 - t] = excl;
  __syncthreads();
  uint32_t above = sh_sum[t];
  if (above < need && need <= above + sum) {
    uint32_t cum = above;
    for (int i = per - 1; i >= 0; --i) {
      if (cum + local[i] >= need) {
        sh_res[0] = t * per + i;
        sh_res[1] = cum;
        break;
      }
      cum += local[i];
    }
  }
  __syncthreads();
  *out_bin = sh_res[0];
  *out_above = sh_res[1];
  __syncthreads();
}

// ------------------------------------------------------------------ 1. sample
__global__ void __launch_bounds__(1024) dgc_sample_kernel(const SegH1* __restrict__ segs) {
  __shared__ uint32_t keys[kSample];
  const SegH1 S = segs[blockIdx.x];
  const uint32_t n = S.n;
  const float* g = seg_g(S);
  const bool exact = n <= (uint32_t)kSample;
  const uint32_t s = exact ? n : (uint32_t)kSample;
  uint32_t p2 = 1;
  while (p2 < s) p2 <<= 1;
  for (uint32_t j = threadIdx.x; j < p2; j += blockDim.x) {
    uint32_t key = 0;
    if (j < s) {
      uint32_t pos;
      if (exact) {
        pos = j;
      } else {
        uint64_t a = (uint64_t)j * n / s, b = (uint64_t)(j + 1) * n / s;
        pos = (uint32_t)(a + splitmix64(S.hash ^ j) % (b - a));
      }
      float acc = S.ef ? __fadd_rn(g[pos], S.r[pos]) : g[pos];
      key = fkey(acc);
    }
    keys[j] = key;
  }
  __syncthreads();
  // bitonic sort, descending
  for (uint32_t size = 2; size <= p2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < p2 / 2; i += blockDim.x) {
        uint32_t lo = 2 * i - (i & (stride - 1));
        uint32_t hi = lo + stride;
        bool desc = ((lo & size) == 0);
        uint32_t a = keys[lo], b = keys[hi];
        if ((a < b) == desc) { keys[lo] = b; keys[hi] = a; }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    uint32_t jstar;
    if (exact) {
      jstar = S.k;
    } else {
      double rs = S.ratio * (double)s;
      double js = ceil(rs + 4.0 * sqrt(rs));
      jstar = js >= (double)s ? s : (uint32_t)js;
      if (jstar < 1) jstar = 1;
    }
    S.st->thr = keys[jstar - 1];
  }
}

// ------------------------------------------------------------------ 2/3. stream
template <bool FALLBACK>
__global__ void __launch_bounds__(kThreads) dgc_stream_kernel(const SegH1* __restrict__ segs,
                                                              const uint32_t* __restrict__ unit_seg) {
  __shared__ uint32_t sh_hist[2048];
  __shared__ uint32_t sh_scan[300];
  __shared__ uint32_t sh_total;
  __shared__ int sh_flag;
  const uint32_t sid = unit_seg[blockIdx.x];
  const SegH1 S = segs[sid];
  if (FALLBACK && *(volatile uint32_t*)&S.st->fallback == 0) return;
  const uint32_t u = blockIdx.x - S.unit0;
  const uint32_t n = S.n;
  for (int i = threadIdx.x; i < 2048; i += kThreads) sh_hist[i] = 0;
  if (threadIdx.x == 0) sh_total = 0;
  __syncthreads();
  const uint32_t thr = FALLBACK ? 0u : S.st->thr;
  const float* g = seg_g(S);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t run = u * (kUnit / kRun) + warp;
  const uint32_t base = run * kRun;
  uint32_t wcount = 0;
  if (base < n) {
    float4 av[8];
    if (FALLBACK) {
      const float* src = S.ef ? S.r : g;
#pragma unroll
      for (int j = 0; j < 8; ++j) av[j] = load4_guard(src, base + j * 128 + lane * 4, n);
    } else {
      float4 gv[8], rv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) gv[j] = load4_stream_guard(g, base + j * 128 + lane * 4, n);
      if (S.ef) {
#pragma unroll
        for (int j = 0; j < 8; ++j) rv[j] = load4_guard(S.r, base + j * 128 + lane * 4, n);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          av[j].x = __fadd_rn(gv[j].x, rv[j].x);
          av[j].y = __fadd_rn(gv[j].y, rv[j].y);
          av[j].z = __fadd_rn(gv[j].z, rv[j].z);
          av[j].w = __fadd_rn(gv[j].w, rv[j].w);
          store4_guard(S.r, base + j * 128 + lane * 4, n, av[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) av[j] = gv[j];
      }
    }
    uint2* cand = S.cand + (size_t)run * kRun;
    const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t e = base + j * 128 + lane * 4;
      uint32_t f[4], bal[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float x = f4get(av[j], c);
        f[c] = (e + c < n) && (fkey(x) >= thr);
        bal[c] = __ballot_sync(0xffffffffu, f[c]);
      }
      uint32_t pre = 0, tot = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        pre += __popc(bal[c] & lt_mask);
        tot += __popc(bal[c]);
      }
      uint32_t pos = wcount + pre;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (f[c]) {
          float x = f4get(av[j], c);
          cand[pos] = make_uint2(e + c, __float_as_uint(x));
          atomicAdd(&sh_hist[fkey(x) >> 20], 1u);
          ++pos;
        }
      }
      wcount += tot;
    }
    if (lane == 0) {
      S.runcnt[run] = wcount;
      atomicAdd(&sh_total, wcount);
    }
  }
  __syncthreads();
  uint32_t* ghist = S.hist + (FALLBACK ? 2048 : 0);
  for (int i = threadIdx.x; i < 2048; i += kThreads) {
    uint32_t h = sh_hist[i];
    if (h) atomicAdd(&ghist[i], h);
  }
  uint32_t* gcount = FALLBACK ? &S.st->count_fb : &S.st->count;
  if (threadIdx.x == 0 && sh_total) atomicAdd(gcount, sh_total);
  if (!last_cta(FALLBACK ? &S.st->done_fb : &S.st->done, S.nunits, &sh_flag)) return;
  const uint32_t total = __ldcg(gcount);
  if (!FALLBACK && total < S.k) {
    if (threadIdx.x == 0) S.st->fallback = 1;
    return;
  }
  uint32_t bin, above;
  select_bin(ghist, 2048, S.k, &bin, &above, sh_scan);
  if (threadIdx.x == 0) {
    S.st->prefix = bin;
    S.st->above = above;
    S.st->need = S.k - above;
  }
}

// ------------------------------------------------------------------ 4. refine
template <int ROUND>
__global__ void __launch_bounds__(kThreads) dgc_refine_kernel(const SegH1* __restrict__ segs,
                                                              const uint32_t* __restrict__ group_seg) {
  __shared__ uint32_t sh_hist[1024];
  __shared__ uint32_t sh_scan[300];
  __shared__ int sh_flag;
  constexpr int kShiftMatch = ROUND == 2 ? 20 : 10;
  constexpr int kShiftBin = ROUND == 2 ? 10 : 0;
  const uint32_t sid = group_seg[blockIdx.x];
  const SegH1 S = segs[sid];
  const uint32_t g = blockIdx.x - S.group0;
  const uint32_t prefix = __ldcg(&S.st->prefix);
  for (int i = threadIdx.x; i < 1024; i += kThreads) sh_hist[i] = 0;
  __syncthreads();
  const uint32_t nruns = (S.n + kRun - 1) / kRun;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t rr = warp; rr < (uint32_t)kRunsPerGroup; rr += kThreads / 32) {
    const uint32_t run = g * kRunsPerGroup + rr;
    if (run >= nruns) break;
    const uint32_t cnt = __ldcg(S.runcnt + run);
    const uint2* cand = S.cand + (size_t)run * kRun;
    for (uint32_t i = lane; i < cnt; i += 32) {
      uint32_t key = __ldcg(&cand[i].y) & 0x7FFFFFFFu;
      if ((key >> kShiftMatch) == prefix) atomicAdd(&sh_hist[(key >> kShiftBin) & 1023u], 1u);
    }
  }
  __syncthreads();
  uint32_t* ghist = S.hist + (ROUND == 2 ? 4096 : 5120);
  for (int i = threadIdx.x; i < 1024; i += kThreads) {
    uint32_t h = sh_hist[i];
    if (h) atomicAdd(&ghist[i], h);
  }
  if (!last_cta(ROUND == 2 ? &S.st->done_r2 : &S.st->done_r3, S.ngroups, &sh_flag)) return;
  const uint32_t need = __ldcg(&S.st->need);
  uint32_t bin, above;
  select_bin(ghist, 1024, need, &bin, &above, sh_scan);
  if (threadIdx.x == 0) {
    S.st->prefix = (prefix << 10) | bin;
    S.st->above = __ldcg(&S.st->above) + above;
    S.st->need = need - above;
  }
}

// ------------------------------------------------------------------ 5. count
__global__ void __launch_bounds__(kThreads) dgc_count_kernel(const SegH1* __restrict__ segs,
                                                             const uint32_t* __restrict__ group_seg) {
  __shared__ uint32_t sh_scan[16];
  __shared__ int sh_flag;
  const uint32_t sid = group_seg[blockIdx.x];
  const SegH1 S = segs[sid];
  const uint32_t g = blockIdx.x - S.group0;
  const uint32_t T = __ldcg(&S.st->prefix);
  const uint32_t nruns = (S.n + kRun - 1) / kRun;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t above = 0, tie = 0;
  for (uint32_t rr = warp; rr < (uint32_t)kRunsPerGroup; rr += kThreads / 32) {
    const uint32_t run = g * kRunsPerGroup + rr;
    if (run >= nruns) break;
    const uint32_t cnt = __ldcg(S.runcnt + run);
    const uint2* cand = S.cand + (size_t)run * kRun;
    for (uint32_t i = lane; i < cnt; i += 32) {
      uint32_t key = __ldcg(&cand[i].y) & 0x7FFFFFFFu;
      above += key > T;
      tie += key == T;
    }
  }
  above = block_sum_u32(above, sh_scan);
  tie = block_sum_u32(tie, sh_scan);
  if (threadIdx.x == 0) {
    S.gcnt[4 * g + 0] = above;
    S.gcnt[4 * g + 1] = tie;
  }
  if (!last_cta(&S.st->done_cnt, S.ngroups, &sh_flag)) return;
  // scan over this segment's groups: tie offsets, then selected offsets
  const uint32_t need = __ldcg(&S.st->need);
  uint32_t tie_carry = 0, sel_carry = 0;
  for (uint32_t g0 = 0; g0 < S.ngroups; g0 += kThreads) {
    const uint32_t gi = g0 + threadIdx.x;
    uint32_t a = 0, t = 0;
    if (gi < S.ngroups) {
      a = __ldcg(&S.gcnt[4 * gi + 0]);
      t = __ldcg(&S.gcnt[4 * gi + 1]);
    }
    uint32_t ttot, stot;
    uint32_t toff = tie_carry + block_excl_scan(t, &ttot, sh_scan);
    uint32_t take = toff >= need ? 0u : min(t, need - toff);
    uint32_t sel = a + take;
    uint32_t soff = sel_carry + block_excl_scan(sel, &stot, sh_scan);
    if (gi < S.ngroups) {
      S.gcnt[4 * gi + 2] = toff;
      S.gcnt[4 * gi + 3] = soff;
    }
    tie_carry += ttot;
    sel_carry += stot;
  }
  if (threadIdx.x == 0) S.st->total_sel = sel_carry;
}

// ------------------------------------------------------------------ 6. write
__global__ void __launch_bounds__(kThreads) dgc_write_kernel(const SegH1* __restrict__ segs,
                                                             const uint32_t* __restrict__ group_seg) {
  __shared__ uint32_t sh_scan[16];
  __shared__ uint32_t sh_off[kRunsPerGroup + 1];
  const uint32_t sid = group_seg[blockIdx.x];
  const SegH1 S = segs[sid];
  const uint32_t g = blockIdx.x - S.group0;
  const uint32_t T = __ldcg(&S.st->prefix);
  const uint32_t need = __ldcg(&S.st->need);
  const uint32_t nruns = (S.n + kRun - 1) / kRun;
  const uint32_t run0 = g * kRunsPerGroup;
  const uint32_t nr = min((uint32_t)kRunsPerGroup, nruns - run0);
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (uint32_t i = 0; i < nr; ++i) {
      sh_off[i] = acc;
      acc += __ldcg(S.runcnt + run0 + i);
    }
    sh_off[nr] = acc;
  }
  __syncthreads();
  const uint32_t C = sh_off[nr];
  uint32_t tie_run = __ldcg(&S.gcnt[4 * g + 2]);
  uint32_t sel_run = __ldcg(&S.gcnt[4 * g + 3]);
  uint32_t* out_idx = reinterpret_cast<uint32_t*>(S.chunk);
  float* out_val = reinterpret_cast<float*>(S.chunk + 4 * (size_t)S.kpad);
  for (uint32_t q0 = 0; q0 < C; q0 += kThreads) {
    const uint32_t q = q0 + threadIdx.x;
    uint32_t is_tie = 0, is_above = 0;
    uint2 c = make_uint2(0, 0);
    if (q < C) {
      uint32_t i = 0;
      while (sh_off[i + 1] <= q) ++i;
      c = __ldcg(S.cand + (size_t)(run0 + i) * kRun + (q - sh_off[i]));
      uint32_t key = c.y & 0x7FFFFFFFu;
      is_above = key > T;
      is_tie = key == T;
    }
    uint32_t ttot;
    uint32_t trank = tie_run + block_excl_scan(is_tie, &ttot, sh_scan);
    uint32_t sel = is_above || (is_tie && trank < need);
    uint32_t stot;
    uint32_t pos = sel_run + block_excl_scan(sel, &stot, sh_scan);
    if (sel) {
      out_idx[pos] = c.x;
      out_val[pos] = __uint_as_float(c.y);
      if (S.ef) S.r[c.x] = 0.0f;
    }
    tie_run += ttot;
    sel_run += stot;
  }
}

// ------------------------------------------------------------------ launchers
void launch_dgc_h1(const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits,
                   const uint32_t* group_seg, int ngroups, cudaStream_t st, cudaEvent_t probe0,
                   cudaEvent_t probe1) {
  if (nsegs == 0) return;
  dgc_sample_kernel<<<nsegs, 1024, 0, st>>>(segs);
  if (probe0) cudaEventRecord(probe0, st);
  dgc_stream_kernel<false><<<nunits, kThreads, 0, st>>>(segs, unit_seg);
  if (probe1) cudaEventRecord(probe1, st);
  dgc_stream_kernel<true><<<nunits, kThreads, 0, st>>>(segs, unit_seg);
  dgc_refine_kernel<2><<<ngroups, kThreads, 0, st>>>(segs, group_seg);
  dgc_refine_kernel<3><<<ngroups, kThreads, 0, st>>>(segs, group_seg);
  dgc_count_kernel<<<ngroups, kThreads, 0, st>>>(segs, group_seg);
  dgc_write_kernel<<<ngroups, kThreads, 0, st>>>(segs, group_seg);
  count_launches(7);
}

}  // namespace esp
