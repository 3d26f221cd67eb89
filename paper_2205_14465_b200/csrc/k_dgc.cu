// DGC / top-k h1 on sm_100a: EF-fused sampled-threshold top-k with index
// compaction (DGC is cited at
// P:828 and evaluated at a 1% rate; EF at P:1427).
//
// Pipeline per bucket (every kernel walks a multi-segment table):
//   1. dgc_sample   one CTA per segment: thr = lower edge of the 21-bit radix bin
//                   holding the j*-th largest key of a hashed stratified sample of
//                   acc = g + r (the k-th key's bin when the whole segment fits the
//                   sample).  Only an accelerator: the result cannot depend on thr
//                   (reading R3); too high a threshold triggers the fallback.
//   2. dgc_stream   ONE persistent, warp-specialised pass over g and r (12 B/elem):
//                   a producer warp streams 16 KB tiles of g and of r into a 4-stage
//                   shared-memory ring with 1D TMA bulk copies (cp.async.bulk +
//                   mbarrier); 8 consumer warps compute acc = g + r, write r := acc,
//                   compact candidates key(acc) >= thr per 512-element run in index
//                   order (vote/ballot/popc) and histogram their top 11 key bits.  The
//                   CTA that completes a segment picks the radix bin of the k-th key.
//                   (TOPK: no threshold; every key is histogrammed, nothing emitted,
//                   and step 3 recompacts from the k-th key's bin up.)
//   3. dgc_fallback only segments with < k candidates: recompact with the
//                   sample's far lower threshold thr_lo (then, if that misses too, 0).
//   4. dgc_refine   two more radix rounds over the candidates -> the exact k-th key
//                   T, #above, #ties to take (ties broken by ascending index).
//   5. dgc_write    per group of runs: count, decoupled look-back for the group's
//                   output offset, ordered selection -> payload idx[]/val[] sorted
//                   by index; EF: r[idx] := 0.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "esp_device.cuh"
#include "esp_internal.h"
#include "esp_kernels.h"

namespace esp {


// CTA-wide (256 threads): find bin b (scanning from the top) with
// above(b) < need <= above(b) + hist[b].  nbins in {1024, 2048}.  GLOBAL: the
// histogram lives in global memory and was built by other CTAs' atomics.
template <int BAR, bool GLOBAL>
__device__ void select_bin(const uint32_t* hist, int nbins, uint32_t need, uint32_t* out_bin,
                           uint32_t* out_above, uint32_t* sh /* >= 270 */, uint32_t* out_total = nullptr) {
  const int per = nbins / kThreads;
  const int t = ctid<BAR>();
  uint32_t local[8];
  uint32_t sum = 0;
  for (int i = 0; i < per; ++i) {
    local[i] = GLOBAL ? __ldcg(hist + t * per + i) : hist[t * per + i];
    sum += local[i];
  }
  uint32_t* sh_sum = sh;        // 256
  uint32_t* sh_res = sh + 256;  // bin, above
  sh_sum[t] = sum;
  csync<BAR>();
  const uint32_t v = sh_sum[kThreads - 1 - t];
  csync<BAR>();
  uint32_t tot;
  const uint32_t excl = block_excl_scan<BAR>(v, &tot, sh + 258);   // sum over threads > (255 - t)
  if (out_total) *out_total = tot;
  sh_sum[kThreads - 1 - t] = excl;
  if (t == 0) { sh_res[0] = 0; sh_res[1] = 0; }
  csync<BAR>();
  const uint32_t above = sh_sum[t];
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
  csync<BAR>();
  *out_bin = sh_res[0];
  *out_above = sh_res[1];
  csync<BAR>();
}

// ------------------------------------------------------------------ 1. sample
// force (test hook, ESP_DGC_FORCE_FALLBACK): bit 0 sets thr above every key so
// that every segment with k > 0 takes the fallback; bit 1 does the same to thr_lo
__global__ void __launch_bounds__(kThreads) dgc_sample_kernel(const SegH1* __restrict__ segs, int force,
                                                             float margin) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  __shared__ uint32_t keys[kSample];
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t sh[280];
  const SegH1 S = segs[blockIdx.x];
  if (S.unsampled) {   // TOPK: no candidates in the streaming pass, which
    if (threadIdx.x == 0) S.st->thr = 0xFFFFFFFFu;   // histograms every key instead
    return;
  }
  const uint32_t n = S.n;
  const float* g = seg_g(S);
  const bool exact = n <= (uint32_t)kSample;
  const uint32_t strata = S.strata;                     // R22: strata of 8 samples
  const uint32_t s = exact ? n : 8u * strata;
  {
    // all 2 x 16 loads of a thread are issued before any is consumed (latency-bound kernel)
    constexpr int kPer = kSample / kThreads;
    float gv[kPer], rv[kPer], uv[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t j = threadIdx.x + q * kThreads;
      uint32_t pos = j;
      if (!exact && j < s) {
        // strata [GN/S, (G+1)N/S), 8 consecutive samples from each at a hashed
        // offset: a random 4-byte gather costs a whole DRAM sector, a run of 8
        // costs one or two (exact mode: a sampler only, the selection stays
        // exact whatever threshold it yields; approximate mode: R22)
        static_assert(kSample == 4096, "512 strata x 8 assumes kSample == 2^12");
        const uint32_t G = j >> 3;
        // (512 strata, the default: shifts instead of 64-bit divisions)
        const uint32_t a = strata == 512 ? (uint32_t)(((uint64_t)G * n) >> 9) : (uint32_t)(((uint64_t)G * n) / strata);
        const uint32_t b = strata == 512 ? (uint32_t)(((uint64_t)(G + 1) * n) >> 9)
                                         : (uint32_t)(((uint64_t)(G + 1) * n) / strata);
        pos = a + (uint32_t)(((uint64_t)(uint32_t)splitmix64(S.hash ^ G) * (b - a - 7)) >> 32) + (j & 7u);
      }
      gv[q] = j < s ? __ldg(g + pos) : 0.f;
      rv[q] = (j < s && S.ef) ? S.r[pos] : 0.f;
      uv[q] = (j < s && S.mom) ? S.mom[pos] : 0.f;
    }
    if (S.mom) {   // momentum correction (R20): the candidate is fl(fl(m u) + g) + v
#pragma unroll
      for (int q = 0; q < kPer; ++q) gv[q] = __fadd_rn(__fmul_rn(S.mcoef, uv[q]), gv[q]);
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t j = threadIdx.x + q * kThreads;
      if (j < s) keys[j] = fkey(S.ef ? __fadd_rn(gv[q], rv[q]) : gv[q]);
    }
  }
  for (int i = threadIdx.x; i < 2048; i += kThreads) hist[i] = 0;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < s; j += kThreads) atomicAdd(&hist[keys[j] >> 20], 1u);
  __syncthreads();
  uint32_t need;
  if (exact) {
    need = S.k;
  } else {
    const double rs = S.ratio * (double)s;
    // exact mode: over-sampled rank (>= k pass w.h.p.); approximate mode: the
    // expected rank of the k-th key (R22)
    const double js = S.approx ? floor(rs + 0.5) : ceil(rs + (double)margin * sqrt(rs));
    need = js >= (double)s ? s : (uint32_t)js;
    if (need < 1) need = 1;
  }
  uint32_t b1, a1, b2, a2;
  select_bin<0, false>(hist, 2048, need, &b1, &a1, sh);
  // the fallback's threshold: the 11-bit bin of a sample rank about twice as
  // deep (a miss at thr is a ~1e-4 event per segment, one at thr_lo needs
  // both tails at once)
  uint32_t b_lo = 0, a_lo;
  if (!exact) select_bin<0, false>(hist, 2048, min(s, 2 * need + 16), &b_lo, &a_lo, sh);
  for (int i = threadIdx.x; i < 1024; i += kThreads) hist[i] = 0;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < s; j += kThreads)
    if ((keys[j] >> 20) == b1) atomicAdd(&hist[(keys[j] >> 10) & 1023u], 1u);
  __syncthreads();
  select_bin<0, false>(hist, 1024, need - a1, &b2, &a2, sh);
  if (threadIdx.x == 0) {
    S.st->thr = (force & 1) ? 0xFFFFFFFFu : (b1 << 20) | (b2 << 10);
    S.st->thr_lo = (force & 2) ? 0xFFFFFFFFu : exact ? 0u : b_lo << 20;
  }
}

// ------------------------------------------------------------------ candidate emission
// One warp, one 1024-element run held in registers (8 float4 per lane; element
// base + j*128 + lane*4 + c).  Appends {idx, bits(acc)} of key >= thr in index
// order and histograms the candidates' top 11 key bits.  Returns the count.
__device__ __forceinline__ uint32_t emit_run(const float4 (&av)[kNJ], uint32_t base, uint32_t n, uint32_t thr,
                                             uint2* __restrict__ cand, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t wcount = 0;
#pragma unroll
  for (int j = 0; j < kNJ; ++j) {
    const uint32_t e = base + j * 128 + lane * 4;
    uint32_t f[4], bal[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      f[c] = (e + c < n) && (fkey(f4get(av[j], c)) >= thr);
      bal[c] = __ballot_sync(0xffffffffu, f[c]);
    }
    if ((bal[0] | bal[1] | bal[2] | bal[3]) == 0) continue;
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
        const float x = f4get(av[j], c);
        cand[pos] = make_uint2(e + c, __float_as_uint(x));
        atomicAdd(&hist[fkey(x) >> 20], 1u);
        ++pos;
      }
    }
    wcount += tot;
  }
  return wcount;
}

// emit_run for a run entirely inside its segment: no bounds tests, and one warp
// vote per float4 column instead of four when nothing passes (~99.7% of them).
__device__ __forceinline__ uint32_t emit_run_full(const float4 (&av)[kNJ], uint32_t base, uint32_t thr,
                                                  uint2* __restrict__ cand, uint32_t* hist) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t wcount = 0;
#pragma unroll
  for (int j = 0; j < kNJ; ++j) {
    const uint32_t f0 = fkey(av[j].x) >= thr, f1 = fkey(av[j].y) >= thr;
    const uint32_t f2 = fkey(av[j].z) >= thr, f3 = fkey(av[j].w) >= thr;
    if (!__any_sync(0xffffffffu, f0 | f1 | f2 | f3)) continue;
    const uint32_t f[4] = {f0, f1, f2, f3};
    uint32_t bal[4], pre = 0, tot = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      bal[c] = __ballot_sync(0xffffffffu, f[c]);
      pre += __popc(bal[c] & lt_mask);
      tot += __popc(bal[c]);
    }
    const uint32_t e = base + j * 128 + lane * 4;
    uint32_t pos = wcount + pre;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (f[c]) {
        const float x = f4get(av[j], c);
        cand[pos] = make_uint2(e + c, __float_as_uint(x));
        atomicAdd(&hist[fkey(x) >> 20], 1u);
        ++pos;
      }
    }
    wcount += tot;
  }
  return wcount;
}

// ------------------------------------------------------------------ 2. stream (TMA)
constexpr int kMaxStages = 6;   // 6 x 32 KB stages + header fit the 227 KB of one SM
constexpr int kMaxGroups = 3;   // consumer groups of 8 warps (tiles in flight being computed)
struct GroupSmem {   // per consumer group
  uint32_t hist[2048];
  uint32_t scan[280];
  uint32_t cta_count;
  int flag;
};
struct StreamSmem {   // followed (128-byte aligned) by `ns` stages of {g[kDgcTile], r[kDgcTile]}
  uint64_t full[kMaxStages], empty[kMaxStages];
  GroupSmem grp[kMaxGroups];
};
constexpr size_t kStreamHdr = (sizeof(StreamSmem) + 127) / 128 * 128;
// a stage: g and r tiles, then the tile's deferred-zeroing record (kZRecMax uint16)
constexpr size_t kStageBytes = 2 * kDgcTile * sizeof(float) + kZRecMax * 2;
// momentum correction (R20): a third tile per stage holds u
constexpr size_t kStageBytesMom = 3 * kDgcTile * sizeof(float) + kZRecMax * 2;
constexpr int kMaxStagesMom = 4;   // 4 x 48 KB + header
template <bool MOM = false>
__device__ __forceinline__ float* stage_g(unsigned char* smem, int s) {
  return reinterpret_cast<float*>(smem + kStreamHdr + (size_t)s * (MOM ? kStageBytesMom : kStageBytes));
}
template <bool MOM = false>
__device__ __forceinline__ float* stage_r(unsigned char* smem, int s) { return stage_g<MOM>(smem, s) + kDgcTile; }
template <bool MOM = false>
__device__ __forceinline__ float* stage_u(unsigned char* smem, int s) { return stage_g<MOM>(smem, s) + 2 * kDgcTile; }
template <bool MOM = false>
__device__ __forceinline__ uint16_t* stage_z(unsigned char* smem, int s) {
  return reinterpret_cast<uint16_t*>(stage_g<MOM>(smem, s) + (MOM ? 3 : 2) * kDgcTile);
}

// segment bookkeeping by the 256 consumer threads of a CTA that has finished its
// share (`units` units) of segment S: flush the private histogram, add the
// candidate count, and if this completes the segment pick the k-th key's bin.
template <int BAR>
__device__ void stream_segment_done(const SegH1& S, uint32_t units, GroupSmem& sm) {
  const int tid = ctid<BAR>();
  csync<BAR>();
  if (units == S.nunits) {
    // the CTA streamed the whole segment: select from its private histogram
    const uint32_t total = sm.cta_count;
    if (S.unsampled) {
      // TOPK: the histogram holds every key and nothing was emitted; the
      // recompaction pass takes the keys from the k-th key's 11-bit bin up
      uint32_t bin, above;
      select_bin<BAR, false>(sm.hist, 2048, S.k, &bin, &above, sm.scan);
      if (tid == 0) {
        S.st->thr_lo = bin << 20;
        S.st->fallback = 1;
        atomicAdd(S.bflag, 1u);
      }
    } else if (total < S.k && !S.approx) {
      if (tid == 0) {
        S.st->fallback = 1;
        atomicAdd(S.bflag, 1u);
      }
    } else {
      // approximate mode with fewer than k candidates: all of them (R22)
      const uint32_t keff = min(total, S.k);
      uint32_t bin, above;
      select_bin<BAR, false>(sm.hist, 2048, keff, &bin, &above, sm.scan);
      if (tid == 0) {
        S.st->prefix = bin;
        S.st->above = above;
        S.st->need = keff - above;
      }
    }
    csync<BAR>();
    for (int i = tid; i < 2048; i += kThreads) sm.hist[i] = 0;
    if (tid == 0) sm.cta_count = 0;
    csync<BAR>();
    return;
  }
  for (int i = tid; i < 2048; i += kThreads) {
    const uint32_t h = sm.hist[i];
    if (h) {
      atomicAdd(&S.hist[i], h);
      sm.hist[i] = 0;
    }
  }
  if (tid == 0) {
    if (sm.cta_count) atomicAdd(&S.st->count, sm.cta_count);
    sm.cta_count = 0;
    __threadfence();
    const uint32_t old = atomicAdd(&S.st->done, units);
    sm.flag = (old + units == S.nunits);
  }
  csync<BAR>();
  if (!sm.flag) return;
  __threadfence();
  const uint32_t total = __ldcg(&S.st->count);
  if (S.unsampled) {   // TOPK (see above)
    uint32_t bin, above;
    select_bin<BAR, true>(S.hist, 2048, S.k, &bin, &above, sm.scan);
    if (tid == 0) {
      S.st->thr_lo = bin << 20;
      S.st->fallback = 1;
      atomicAdd(S.bflag, 1u);
    }
    return;
  }
  if (total < S.k && !S.approx) {
    if (tid == 0) {
      S.st->fallback = 1;
      atomicAdd(S.bflag, 1u);
    }
    csync<BAR>();
    return;
  }
  const uint32_t keff = min(total, S.k);   // approximate mode: all candidates if fewer than k (R22)
  uint32_t bin, above;
  select_bin<BAR, true>(S.hist, 2048, keff, &bin, &above, sm.scan);
  if (tid == 0) {
    S.st->prefix = bin;
    S.st->above = above;
    S.st->need = keff - above;
  }
}

// NCG consumer groups of 8 warps: group c takes the CTA's tiles i = c, c + NCG,
// ... (stage i mod ns), so NCG tiles are computed at once while the producer
// keeps the ring full.  ns must be a multiple of NCG: then every use of a stage
// by a group follows that group's own previous use of it, which is what makes
// the one-bit phase parity of the full barrier unambiguous (with ns % NCG != 0
// a warp could pass a parity test one fill early).
template <int NCG, bool MOM = false>
__global__ void __launch_bounds__(NCG * kThreads + 32, 1) dgc_stream_kernel(const SegH1* __restrict__ segs,
                                                                            const uint32_t* __restrict__ unit_seg,
                                                                            uint32_t nunits, int ns) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  StreamSmem& sm = *reinterpret_cast<StreamSmem*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t u0 = (uint32_t)((uint64_t)blockIdx.x * nunits / gridDim.x);
  const uint32_t u1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * nunits / gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kThreads / 32);
    }
    fence_barrier_init();
    for (int c = 0; c < NCG; ++c) sm.grp[c].cta_count = 0;
  }
  for (int i = threadIdx.x; i < NCG * 2048; i += blockDim.x) sm.grp[i / 2048].hist[i % 2048] = 0;
  __syncthreads();
  // the prologue above (barrier init, histogram zeroing) overlapped the
  // predecessor's tail (PDL); everything below reads what it wrote
  pdl_wait();
  pdl_trigger();

  if (warp == NCG * kThreads / 32) {
    // ---- producer warp: one elected lane streams tiles into the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      // per-segment values are cached; the unit table is prefetched one ahead
      uint32_t cur = 0xFFFFFFFFu, unit0 = 0, n = 0;
      const float* gseg = nullptr;
      const float* rseg = nullptr;
      const float* useg = nullptr;
      const uint16_t* zseg = nullptr;
      uint32_t zcap = 0;
      bool ef = false;
      uint32_t sid_next = u0 < u1 ? unit_seg[u0] : 0u;
      int stage = 0;
      uint32_t phase = 0;
      bool wrapped = false;
      for (uint32_t u = u0; u < u1; ++u) {
        const uint32_t sid = sid_next;
        if (u + 1 < u1) sid_next = unit_seg[u + 1];
        if (sid != cur) {
          const SegH1& S = segs[sid];
          cur = sid;
          unit0 = S.unit0;
          n = S.n;
          gseg = seg_g(S);
          rseg = S.r;
          useg = S.mom;
          zseg = S.zrec;
          zcap = S.zcap;
          ef = S.ef != 0;
        }
        if (wrapped) mbar_wait(&sm.empty[stage], phase ^ 1);
        const uint32_t start = (u - unit0) * kDgcTile;
        const uint32_t len = min((uint32_t)kDgcTile, n - start);
        const float* g = gseg + start;
        const float* r = rseg + start;
        const float* um = useg + start;
        const uint32_t bytes = (len * 4) & ~15u;
        if (bytes && al16(g) && (!ef || al16(r)) && (!MOM || al16(um))) {
          const uint32_t zb = zseg ? zcap * 2 : 0u;   // the tile's deferred-zeroing record
          mbar_arrive_expect_tx(&sm.full[stage], bytes * ((ef ? 2 : 1) + (MOM ? 1 : 0)) + zb);
          tma_load_1d(stage_g<MOM>(smem_raw, stage), g, bytes, &sm.full[stage], pol);
          if (ef) tma_load_1d(stage_r<MOM>(smem_raw, stage), r, bytes, &sm.full[stage], pol);
          if (MOM) tma_load_1d(stage_u<MOM>(smem_raw, stage), um, bytes, &sm.full[stage], pol);
          if (zb) tma_load_1d(stage_z<MOM>(smem_raw, stage), zseg + (size_t)(u - unit0) * zcap, zb, &sm.full[stage], pol);
        } else {
          mbar_arrive(&sm.full[stage]);
        }
        if (++stage == ns) {
          stage = 0;
          phase ^= 1;
          wrapped = true;
        }
      }
    }
    return;
  }

  // ---- NCG groups of 8 consumer warps
  const int cg = NCG == 1 ? 0 : warp / (kThreads / 32);
  GroupSmem& gs = sm.grp[cg];
  auto seg_done = [&](const SegH1& S, uint32_t units) {
    if (NCG == 1 || cg == 0) stream_segment_done<1>(S, units, gs);
    else if (cg == 1) stream_segment_done<2>(S, units, gs);
    else stream_segment_done<3>(S, units, gs);
  };
  uint32_t cur = 0xFFFFFFFFu, cur_units = 0, thr = 0;
  const float* g = nullptr;
  SegH1 S{};
  uint32_t sid_next = u0 + cg < u1 ? unit_seg[u0 + cg] : 0u;
  int stage = cg;
  uint32_t phase = 0;
  for (uint32_t u = u0 + cg; u < u1; u += NCG) {
    const uint32_t sid = sid_next;
    if (u + NCG < u1) sid_next = unit_seg[u + NCG];
    if (sid != cur) {
      if (cur != 0xFFFFFFFFu) seg_done(S, cur_units);
      cur = sid;
      S = segs[sid];
      g = seg_g(S);
      thr = __ldcg(&S.st->thr);
      cur_units = 0;
    }
    ++cur_units;
    const uint32_t start = (u - S.unit0) * kDgcTile;
    const uint32_t n = S.n;
    const uint32_t lbase = (warp & 7) * kRun;      // tile-relative
    const uint32_t base = start + lbase;           // segment-relative
    // fast path: a whole tile in shared memory (aligned, EF on, inside the segment)
    const bool full = S.ef && start + kDgcTile <= n && al16(g + start) && al16(S.r + start) &&
                      (!MOM || al16(S.mom + start));
    float4 av[kNJ];
    float4 um[MOM ? kNJ : 1];   // MOM: u' = fl(fl(m u) + g), stored after the stage is released
    mbar_wait(&sm.full[stage], phase);
    if (S.zrec) {
      // the previous call's selection in this warp's run reads r = u = +0
      // (deferred EF zeroing: the write kernel recorded it instead of scattering
      // zeros into r); in the staged tile, or in memory for an unstaged one
      const uint32_t len = min((uint32_t)kDgcTile, n - start);
      const uint32_t sb = (len * 4) & ~15u;
      const bool staged = sb && al16(g + start) && (!S.ef || al16(S.r + start)) && (!MOM || al16(S.mom + start));
      const uint16_t* z = staged ? stage_z<MOM>(smem_raw, stage) : S.zrec + (size_t)(u - S.unit0) * S.zcap;
      const uint32_t cnt = min((uint32_t)z[0], S.zcap - 1);
      bool wrote = false;
      for (uint32_t i = 1 + lane; i <= cnt; i += 32) {
        const uint32_t off = z[i];
        if (off - lbase >= (uint32_t)kRun || start + off >= n) continue;   // another warp's run
        if (staged && off < sb / 4) {
          if (S.ef) stage_r<MOM>(smem_raw, stage)[off] = 0.f;
          if (MOM) stage_u<MOM>(smem_raw, stage)[off] = 0.f;
          wrote = true;
        } else {
          if (S.ef) S.r[start + off] = 0.f;
          if (MOM) S.mom[start + off] = 0.f;
        }
      }
      if (wrote) fence_proxy_async_smem();   // generic writes into a TMA stage before its reuse
      __syncwarp();
    }
    if (full) {
      const float* sg = stage_g<MOM>(smem_raw, stage) + lbase + lane * 4;
      const float* sr = stage_r<MOM>(smem_raw, stage) + lbase + lane * 4;
#pragma unroll
      for (int j = 0; j < kNJ; ++j) {
        float4 gv = lds4(sg + j * 128);
        const float4 rv = lds4(sr + j * 128);
        if (MOM) {
          const float4 uv = lds4(stage_u<MOM>(smem_raw, stage) + lbase + lane * 4 + j * 128);
          gv.x = __fadd_rn(__fmul_rn(S.mcoef, uv.x), gv.x);
          gv.y = __fadd_rn(__fmul_rn(S.mcoef, uv.y), gv.y);
          gv.z = __fadd_rn(__fmul_rn(S.mcoef, uv.z), gv.z);
          gv.w = __fadd_rn(__fmul_rn(S.mcoef, uv.w), gv.w);
          um[MOM ? j : 0] = gv;
        }
        av[j].x = __fadd_rn(gv.x, rv.x);
        av[j].y = __fadd_rn(gv.y, rv.y);
        av[j].z = __fadd_rn(gv.z, rv.z);
        av[j].w = __fadd_rn(gv.w, rv.w);
      }
    } else {
      const uint32_t len = min((uint32_t)kDgcTile, n - start);
      const uint32_t bytes = (len * 4) & ~15u;
      const bool tma = bytes && al16(g + start) && (!S.ef || al16(S.r + start)) && (!MOM || al16(S.mom + start));
#pragma unroll
      for (int j = 0; j < kNJ; ++j) {
        const uint32_t l = lbase + j * 128 + lane * 4;
        const uint32_t e = start + l;
        float4 gv, rv;
        if (tma && l + 4 <= bytes / 4) {
          gv = lds4(stage_g<MOM>(smem_raw, stage) + l);
          rv = S.ef ? lds4(stage_r<MOM>(smem_raw, stage) + l) : make_float4(0.f, 0.f, 0.f, 0.f);
          if (MOM) {
            const float4 uv = lds4(stage_u<MOM>(smem_raw, stage) + l);
            gv.x = __fadd_rn(__fmul_rn(S.mcoef, uv.x), gv.x);
            gv.y = __fadd_rn(__fmul_rn(S.mcoef, uv.y), gv.y);
            gv.z = __fadd_rn(__fmul_rn(S.mcoef, uv.z), gv.z);
            gv.w = __fadd_rn(__fmul_rn(S.mcoef, uv.w), gv.w);
          }
        } else {
          gv = load4_guard(g, e, n);
          rv = S.ef ? load4_guard(S.r, e, n) : make_float4(0.f, 0.f, 0.f, 0.f);
          if (MOM) {
            const float4 uv = load4_guard(S.mom, e, n);
            gv.x = __fadd_rn(__fmul_rn(S.mcoef, uv.x), gv.x);
            gv.y = __fadd_rn(__fmul_rn(S.mcoef, uv.y), gv.y);
            gv.z = __fadd_rn(__fmul_rn(S.mcoef, uv.z), gv.z);
            gv.w = __fadd_rn(__fmul_rn(S.mcoef, uv.w), gv.w);
          }
        }
        if (MOM) um[MOM ? j : 0] = gv;
        if (S.ef) {
          av[j].x = __fadd_rn(gv.x, rv.x);
          av[j].y = __fadd_rn(gv.y, rv.y);
          av[j].z = __fadd_rn(gv.z, rv.z);
          av[j].w = __fadd_rn(gv.w, rv.w);
        } else {
          av[j] = gv;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);   // stage consumed (values in registers)
    stage += NCG;
    if (stage >= ns) {
      stage -= ns;
      phase ^= 1;
    }
    if (base < n) {
      if (full) {
        float* rp = S.r + base + lane * 4;
#pragma unroll
        for (int j = 0; j < kNJ; ++j) st4(rp + j * 128, av[j]);
        if (MOM) {
          float* up = S.mom + base + lane * 4;
#pragma unroll
          for (int j = 0; j < kNJ; ++j) st4(up + j * 128, um[MOM ? j : 0]);
        }
      } else if (S.ef) {
#pragma unroll
        for (int j = 0; j < kNJ; ++j) store4_guard(S.r, base + j * 128 + lane * 4, n, av[j]);
        if (MOM) {
#pragma unroll
          for (int j = 0; j < kNJ; ++j) store4_guard(S.mom, base + j * 128 + lane * 4, n, um[MOM ? j : 0]);
        }
      }
      const uint32_t run = base / kRun;
      if (S.unsampled) {
        // TOPK: the top 11 bits of every key (the radix select's first digit)
#pragma unroll
        for (int j = 0; j < kNJ; ++j) {
          const uint32_t e = base + j * 128 + lane * 4;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (e + c < n) atomicAdd(&gs.hist[fkey(f4get(av[j], c)) >> 20], 1u);
        }
      }
      const uint32_t wc = full ? emit_run_full(av, base, thr, S.cand + (size_t)run * kRun, gs.hist)
                               : emit_run(av, base, n, thr, S.cand + (size_t)run * kRun, gs.hist);
      if (lane == 0) {
        S.runcnt[run] = wc;
        if (wc) atomicAdd(&gs.cta_count, wc);
      }
    }
  }
  if (cur != 0xFFFFFFFFu) seg_done(S, cur_units);
}

// ------------------------------------------------------------------ 3. fallback
// Segments whose sampled threshold let fewer than k candidates through are
// recompacted from acc (= r after the streaming pass) with thr_lo.  Every CTA
// scans the segment list; only flagged segments cost work.
__device__ void fallback_pass(const SegH1* __restrict__ segs, int nsegs, uint32_t cta, uint32_t ncta) {
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t sh[280];
  __shared__ uint32_t cta_count;
  __shared__ int flag;
  __shared__ uint32_t list[256];
  __shared__ uint32_t nlist;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (__ldcg(segs[0].bflag) == 0) return;   // no segment of this bucket fell back
  for (int s0 = 0; s0 < nsegs; s0 += kThreads) {
    if (threadIdx.x == 0) nlist = 0;
    __syncthreads();
    if (s0 + threadIdx.x < nsegs && __ldcg(&segs[s0 + threadIdx.x].st->fallback))
      list[atomicAdd(&nlist, 1u)] = s0 + threadIdx.x;
    __syncthreads();
    const uint32_t cnt = nlist;
    for (uint32_t li = 0; li < cnt; ++li) {
    const uint32_t sid = list[li];
    const SegH1 S = segs[sid];
    if (cta >= S.nunits) continue;
    for (int i = threadIdx.x; i < 2048; i += kThreads) hist[i] = 0;
    if (threadIdx.x == 0) cta_count = 0;
    __syncthreads();
    uint32_t units = 0;
    const float* src = S.ef ? S.r : seg_g(S);
    const uint32_t thr_fb = __ldcg(&S.st->thr_lo);
    auto recompact = [&](uint32_t u0, uint32_t ustep, uint32_t thr) {
      for (uint32_t u = u0; u < S.nunits; u += ustep, ++units) {
        const uint32_t base = u * kDgcTile + warp * kRun;
        if (base >= S.n) continue;
        float4 av[kNJ];
#pragma unroll
        for (int j = 0; j < kNJ; ++j) av[j] = load4_guard(src, base + j * 128 + lane * 4, S.n);
        const uint32_t run = base / kRun;
        const uint32_t wc = emit_run(av, base, S.n, thr, S.cand + (size_t)run * kRun, hist);
        if (lane == 0) {
          S.runcnt[run] = wc;
          atomicAdd(&cta_count, wc);
        }
      }
    };
    recompact(cta, ncta, thr_fb);
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += kThreads)
      if (hist[i]) atomicAdd(&S.hist[2048 + i], hist[i]);
    if (threadIdx.x == 0) {
      atomicAdd(&S.st->count_fb, cta_count);
      __threadfence();
      const uint32_t old = atomicAdd(&S.st->done_fb, units);
      flag = (old + units == S.nunits);
    }
    __syncthreads();
    if (flag) {
      __threadfence();
      if (__ldcg(&S.st->count_fb) < S.k) {
        // thr_lo missed as well (both sample tails at once): this CTA alone
        // recompacts the whole segment with thr = 0 -- slow, and never expected
        __syncthreads();
        for (int i = threadIdx.x; i < 2048; i += kThreads) {
          hist[i] = 0;
          S.hist[2048 + i] = 0;
        }
        __syncthreads();
        recompact(0, 1, 0u);
        __syncthreads();
        for (int i = threadIdx.x; i < 2048; i += kThreads) S.hist[2048 + i] = hist[i];
        __threadfence();
        __syncthreads();
      }
      uint32_t bin, above;
      select_bin<0, true>(S.hist + 2048, 2048, S.k, &bin, &above, sh);
      if (threadIdx.x == 0) {
        S.st->prefix = bin;
        S.st->above = above;
        S.st->need = S.k - above;
      }
    }
    __syncthreads();
    }
  }
}

// Thin kernel over the fallback pass (every CTA scans the segment list).
__global__ void __launch_bounds__(kThreads) dgc_fallback_kernel(const SegH1* __restrict__ segs, int nsegs) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  fallback_pass(segs, nsegs, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------------ 4. refine
// A finalize group = S.rpg (8..128, a power of two) consecutive runs of one
// segment, owned by ONE WARP: the finalize is a chain of dependent small loads
// (descriptor, run counts, candidates, counters), so it is throughput-bound on
// the number of independent chains in flight -- 64 warps per SM, no CTA
// barriers.  The planner sizes rpg so that a group expects about one batch of
// candidates (kBatch x 32): dense candidate segments (1% ratios) get short
// groups, so each warp's chain of dependent candidate loads stays one or two
// round trips long.  The group's candidates are addressed as one flat,
// index-ordered list: off[i] = first flat position of run i (lane l holds
// runs l * ppl .. l * ppl + ppl - 1, ppl = rpg / 32 or 1).  128-run groups
// (0.1% ratios) keep BERT-large's ~5300 groups within one wave of warps.
static_assert(kRunsPerGroup == 128, "at most four run counts per lane");
static_assert(kDgcTile == 4096, "deferred-zeroing records address tiles as idx >> 12");
constexpr int kBatch = 4;   // candidate loads in flight per lane
// refine: a group with up to this many candidates adds its matches to the
// global round histogram directly; larger groups (1% ratios, TOPK, fallbacks)
// count into a warp-private shared histogram flushed once, so that a round
// with millions of matches (a 2^28-element tensor at 1%) costs one atomic per
// (group, non-empty bin) instead of one per match on a few hot bins
constexpr uint32_t kDirect = 64;
constexpr int kSepGroupsPerSeg = 256;   // above this mean, the round selects run as kernels
constexpr int kWarpsPerCta = kThreads / 32;

struct WarpGroup {
  const SegH1* S;
  uint32_t g;      // group index within the segment
  uint32_t C;      // candidates in the group
  uint32_t nr;     // runs in the group
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// off: this warp's 65-entry offset table in shared memory
__device__ __forceinline__ WarpGroup warp_group_offsets(const SegH1* segs, const uint32_t* group_seg, uint32_t gi,
                                                        uint32_t* off) {
  const int lane = threadIdx.x & 31;
  WarpGroup G;
  G.S = segs + group_seg[gi];
  const SegH1& S = *G.S;
  G.g = gi - S.group0;
  const uint32_t nruns = (S.n + kRun - 1) / kRun;
  const uint32_t rpg = S.rpg;
  const uint32_t run0 = G.g * rpg;
  G.nr = min(rpg, nruns - run0);
  const uint32_t ppl = rpg > 32 ? rpg / 32 : 1u;   // runs per lane (1, 2 or 4)
  const uint32_t i0 = ppl * lane;
  uint32_t c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = ((uint32_t)j < ppl && i0 + j < G.nr) ? __ldcg(S.runcnt + run0 + i0 + j) : 0u;
  const uint32_t incl = warp_incl_scan(c[0] + c[1] + c[2] + c[3]);
  uint32_t ex = incl - (c[0] + c[1] + c[2] + c[3]);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if ((uint32_t)j < ppl && i0 + j < rpg) off[i0 + j] = ex;
    ex += c[j];
  }
  G.C = __shfl_sync(0xffffffffu, incl, 31);
  if (lane == 31) off[rpg] = incl;
  __syncwarp();
  return G;
}

__device__ __forceinline__ uint2 warp_group_cand(const WarpGroup& G, const uint32_t* off, uint32_t q) {
  uint32_t lo = 0, hi = G.nr;   // largest i with off[i] <= q
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= q) lo = mid; else hi = mid;
  }
  return __ldcg(G.S->cand + (size_t)(G.g * G.S->rpg + lo) * kRun + (q - off[lo]));
}

// After round 2 a group's candidates are DENSE: compacted in place to the
// front of the group's slot range, the count in runcnt[first run].
__device__ __forceinline__ WarpGroup warp_group_dense(const SegH1* segs, const uint32_t* group_seg, uint32_t gi) {
  WarpGroup G;
  G.S = segs + group_seg[gi];
  G.g = gi - G.S->group0;
  G.nr = 0;
  G.C = __ldcg(G.S->runcnt + (size_t)G.g * G.S->rpg);
  return G;
}
__device__ __forceinline__ uint2* group_slots(const WarpGroup& G) {
  return G.S->cand + (size_t)G.g * G.S->rpg * kRun;
}

// Warp-wide: bin b of a 1024-bin global histogram, the sum of `rep` replicas
// (scanning from the top) with above(b) < need <= above(b) + hist[b]; (0, 0)
// if there is none (as select_bin).
__device__ __forceinline__ void warp_select_bin(const uint32_t* hist, uint32_t rep, uint32_t need,
                                                uint32_t* out_bin, uint32_t* out_above) {
  const int lane = threadIdx.x & 31;
  // a lane's 32 bins as 4 chunk sums of 8 (no 32-entry array: the refine
  // kernels run at 32 registers); the selected lane reloads one chunk
  uint32_t cs[4] = {0u, 0u, 0u, 0u};
  for (uint32_t r = 0; r < rep; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(hist + 1024u * r) + lane * 8 + i);
      cs[i >> 1] += v.x + v.y + v.z + v.w;
    }
  }
  const uint32_t sum = cs[0] + cs[1] + cs[2] + cs[3];
  // above this lane's bins = sum over lanes > lane (suffix scan)
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, x, o);
    if (lane + o < 32) x += y;
  }
  const uint32_t above = x - sum;
  uint32_t bin = 0, ab = 0;
  const bool mine = above < need && need <= above + sum;
  if (mine) {   // the chunk holding the bin (from the top), then its 8 bins
    uint32_t cum = above;
    int c = 3;
#pragma unroll
    for (int q = 3; q > 0; --q)
      if (c == q && cum + cs[q] < need) {
        cum += cs[q];
        c = q - 1;
      }
    uint32_t h8[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    for (uint32_t r = 0; r < rep; ++r) {
      const uint4* p = reinterpret_cast<const uint4*>(hist + 1024u * r + lane * 32 + 8 * c);
      const uint4 a = __ldcg(p), b = __ldcg(p + 1);
      h8[0] += a.x; h8[1] += a.y; h8[2] += a.z; h8[3] += a.w;
      h8[4] += b.x; h8[5] += b.y; h8[6] += b.z; h8[7] += b.w;
    }
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      if (cum + h8[i] >= need) { bin = lane * 32 + 8 * c + i; ab = cum; break; }
      cum += h8[i];
    }
  }
  const uint32_t m = __ballot_sync(0xffffffffu, mine);
  if (m) {
    const int src = __ffs(m) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    ab = __shfl_sync(0xffffffffu, ab, src);
  }
  *out_bin = m ? bin : 0u;
  *out_above = m ? ab : 0u;
}

// LAST: the warp that completes a segment's round (fence + counter) selects
// the next 10 bits; else dgc_select_kernel does it after the kernel (segments
// with thousands of groups: one contended counter and a fence per warp cost
// more than a launch)
template <int ROUND, bool LAST>
__global__ void __launch_bounds__(kThreads, 6) dgc_refine_kernel(const SegH1* __restrict__ segs,
                                                              const uint32_t* __restrict__ group_seg,
                                                              uint32_t ngroups) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  __shared__ uint32_t sh_off[kWarpsPerCta][kRunsPerGroup + 1];
  // 1024 16-bit bins per warp, two per word (groups of more than 65535
  // candidates count directly in global memory)
  __shared__ uint32_t sh_hist[kWarpsPerCta][512];
  constexpr int kShiftMatch = ROUND == 2 ? 20 : 10;
  constexpr int kShiftBin = ROUND == 2 ? 10 : 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t gi = blockIdx.x * kWarpsPerCta + w;
  if (gi >= ngroups) return;   // warp-uniform; this kernel has no CTA barrier
  uint32_t* off = sh_off[w];
  // round 2 reads the run-major candidates and compacts them in place (every
  // later pass reads them densely); round 3 reads the dense list
  const WarpGroup G = ROUND == 2 ? warp_group_offsets(segs, group_seg, gi, off) : warp_group_dense(segs, group_seg, gi);
  const SegH1& S = *G.S;
  uint2* dense = group_slots(G);
  const uint32_t prefix = __ldcg(&S.st->prefix);
  // this warp's replica of the round histogram
  uint32_t* const ghist_all = S.hist + 4096 + (ROUND == 2 ? 0u : 1024u * S.hrep);
  uint32_t* ghist = ghist_all + 1024u * (G.g % S.hrep);
  // few candidates (the sampled DGC case): global atomics per match; many
  // (TOPK, fallbacks): a warp-private shared histogram, flushed once
  // (16-bit warp bins: a group of 128 runs can hold 65536 candidates)
  const bool direct = G.C <= kDirect || G.C > 0xFFFFu;
  uint32_t* wh = sh_hist[w];
  if (!direct) {
    for (int i = lane; i < 512; i += 32) wh[i] = 0;
    __syncwarp();
  }
  // round 3 also leaves the write kernel a per-group record (in the run-count
  // slots 1..3 of the group, free once round 2 made the list dense): the
  // candidates above the 21-bit bin of T, those inside it, and up to three of
  // their low 10 bits -- enough to count #above / #ties of T without a pass
  uint32_t n_hi = 0, n_in = 0, packed = 0;
  for (uint32_t base = 0; base < G.C; base += kBatch * 32) {   // warp-uniform trip count
    uint2 cv[kBatch];
#pragma unroll
    for (int m = 0; m < kBatch; ++m) {
      const uint32_t q = base + m * 32 + lane;
      cv[m] = q < G.C ? (ROUND == 2 ? warp_group_cand(G, off, q) : __ldcg(dense + q)) : make_uint2(0u, 0u);
    }
    if (ROUND == 2) {
      // slot q <= the source slot of every candidate >= q, so once the whole
      // batch is in registers its stores clobber nothing unread
      __syncwarp();
#pragma unroll
      for (int m = 0; m < kBatch; ++m) {
        const uint32_t q = base + m * 32 + lane;
        if (q < G.C) dense[q] = cv[m];
      }
    }
#pragma unroll
    for (int m = 0; m < kBatch; ++m) {
      const uint32_t key = cv[m].y & 0x7FFFFFFFu;
      const bool valid = base + m * 32 + lane < G.C;
      const bool match = valid && (key >> kShiftMatch) == prefix;
      if (match) {
        const uint32_t bin = (key >> kShiftBin) & 1023u;
        if (direct) atomicAdd(&ghist[bin], 1u);
        else atomicAdd(&wh[bin >> 1], 1u << (16 * (bin & 1)));
      }
      if (ROUND == 3) {
        n_hi += __popc(__ballot_sync(0xffffffffu, valid && (key >> kShiftMatch) > prefix));
        const uint32_t mb = __ballot_sync(0xffffffffu, match);
        const uint32_t pos = n_in + __popc(mb & ((1u << lane) - 1u));
        packed |= __reduce_or_sync(0xffffffffu, (match && pos < 3) ? (key & 1023u) << (10 * pos) : 0u);
        n_in += __popc(mb);
      }
    }
  }
  if (ROUND == 3 && lane == 0) {
    uint32_t* rec = S.runcnt + (size_t)G.g * S.rpg;
    rec[1] = n_hi;
    rec[2] = n_in;
    rec[3] = packed;
  }
  if (ROUND == 2 && lane == 0) S.runcnt[(size_t)G.g * S.rpg] = G.C;   // the dense count
  if (!direct) {
    __syncwarp();
    for (int i = lane; i < 512; i += 32) {
      const uint32_t h = wh[i];
      if (h & 0xFFFFu) atomicAdd(&ghist[2 * i], h & 0xFFFFu);
      if (h >> 16) atomicAdd(&ghist[2 * i + 1], h >> 16);
    }
  }
  if (!LAST) return;
  // the warp that completes the segment's round selects the next 10 bits
  uint32_t last = 0;
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(ROUND == 2 ? &S.st->done_r2 : &S.st->done_r3, 1u) == S.ngroups - 1;
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  const uint32_t need = __ldcg(&S.st->need);
  uint32_t bin, above;
  warp_select_bin(ghist_all, S.hrep, need, &bin, &above);
  if (lane == 0) {
    S.st->prefix = (prefix << 10) | bin;
    S.st->above = __ldcg(&S.st->above) + above;
    S.st->need = need - above;
  }
}

// The round's bin selection for every segment with finalize groups, one warp
// each, after the refine kernel (the kernel boundary orders the histogram).
template <int ROUND>
__global__ void __launch_bounds__(32) dgc_select_kernel(const SegH1* __restrict__ segs) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  const SegH1& S = segs[blockIdx.x];
  if (S.ngroups == 0) return;
  const uint32_t prefix = __ldcg(&S.st->prefix);
  const uint32_t need = __ldcg(&S.st->need);
  uint32_t bin, above;
  warp_select_bin(S.hist + 4096 + (ROUND == 2 ? 0u : 1024u * S.hrep), S.hrep, need, &bin, &above);
  if (threadIdx.x == 0) {
    S.st->prefix = (prefix << 10) | bin;
    S.st->above = __ldcg(&S.st->above) + above;
    S.st->need = need - above;
  }
}

// ------------------------------------------------------------------ 5. write
// Whether element i of S is one of dgc_sample_kernel's sample positions (the
// same strata and hashed offsets, which do not depend on the step): the next
// call's sampler reads r and u there directly, so a selected sample position is
// zeroed in memory at once instead of only recorded (a few per segment).
__device__ __forceinline__ bool dgc_is_sample(const SegH1& S, uint32_t i) {
  const uint32_t n = S.n, strata = S.strata;
  if (S.unsampled) return false;
  if (n <= (uint32_t)kSample) return true;   // the whole segment is sampled
  auto lo_of = [&](uint32_t G) -> uint32_t {
    return strata == 512 ? (uint32_t)(((uint64_t)G * n) >> 9) : (uint32_t)(((uint64_t)G * n) / strata);
  };
  uint32_t G = (uint32_t)((float)i / (float)n * (float)strata);   // within a few; corrected below
  if (G >= strata) G = strata - 1;
  while (G + 1 < strata && lo_of(G + 1) <= i) ++G;
  while (G > 0 && lo_of(G) > i) --G;
  const uint32_t a = lo_of(G), b = lo_of(G + 1);
  const uint32_t p0 = a + (uint32_t)(((uint64_t)(uint32_t)splitmix64(S.hash ^ G) * (b - a - 7)) >> 32);
  return i >= p0 && i < p0 + 8;
}

// Look-back status word of a group: flag (2 bits: 1 aggregate, 2 inclusive
// prefix, 3 exclusive prefix from dgc_scan_kernel) | #above (31 bits) | #ties (31 bits).
__device__ __forceinline__ unsigned long long lb_pack(uint32_t flag, uint32_t above, uint32_t tie) {
  return ((unsigned long long)flag << 62) | ((unsigned long long)above << 31) | tie;
}

// Every group's output offset when round 3's records cover the whole
// segment (each group has <= 3 candidates inside T's 21-bit bin): one CTA per
// segment scans the groups' (#above, #ties) -- a thread per contiguous run of
// groups, one CTA scan -- and stores each group's EXCLUSIVE prefix (flag 3).
// The write kernel then needs no look-back: the decoupled look-back walks
// 32 groups per round trip, i.e. ~100 us for the 4096 groups of a 2^28-element
// tensor whose aggregates all appear at once.  A segment with a group beyond
// the records (many equal keys) is left to the look-back.
// exclusive scan of (a, t) over the NT threads of a CTA in thread order; sh
// needs 2 x 33 words
template <int NT>
__device__ __forceinline__ uint2 scan_excl2(uint32_t a, uint32_t t, uint32_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t xa = a, xt = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, o), yt = __shfl_up_sync(0xffffffffu, xt, o);
    if (lane >= o) {
      xa += ya;
      xt += yt;
    }
  }
  if (lane == 31) {
    sh[warp] = xa;
    sh[33 + warp] = xt;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t wa = lane < NT / 32 ? sh[lane] : 0u, wt = lane < NT / 32 ? sh[33 + lane] : 0u;
    uint32_t sa = wa, st = wt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ya = __shfl_up_sync(0xffffffffu, sa, o), yt = __shfl_up_sync(0xffffffffu, st, o);
      if (lane >= o) {
        sa += ya;
        st += yt;
      }
    }
    sh[lane] = sa - wa;
    sh[33 + lane] = st - wt;
  }
  __syncthreads();
  return make_uint2(xa - a + sh[warp], xt - t + sh[33 + warp]);
}

// One CTA of NT threads per segment (1024 for segments of thousands of groups,
// else 256); each thread a contiguous run of groups whose 16-byte records
// (count, #above, #inside, packed low bits) are loaded kScanB at a time, all in
// flight together (a 2^28-element tensor at 1%: 4096 groups, one batch per
// thread).
template <int NT>
__global__ void __launch_bounds__(NT) dgc_scan_kernel(const SegH1* __restrict__ segs) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  constexpr int kScanB = 8;
  __shared__ uint32_t sh[66];
  const SegH1& S = segs[blockIdx.x];
  const uint32_t G = S.ngroups;
  if (G == 0) return;
  const uint32_t T = __ldcg(&S.st->prefix), b3 = T & 1023u;
  const uint32_t per = (G + NT - 1) / NT;
  const uint32_t g0 = min(G, threadIdx.x * per), g1 = min(G, g0 + per);
  const uint32_t rpg = S.rpg;
  auto rec_of = [&](uint32_t g) { return __ldcg(reinterpret_cast<const uint4*>(S.runcnt + (size_t)g * rpg)); };
  uint32_t ta = 0, tt = 0;
  bool bad = false;
  for (uint32_t gb = g0; gb < g1; gb += kScanB) {
    uint4 rec[kScanB];
#pragma unroll
    for (int j = 0; j < kScanB; ++j) rec[j] = gb + j < g1 ? rec_of(gb + j) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < kScanB; ++j) {
      ta += rec[j].y;
      bad |= rec[j].z > 3;
#pragma unroll
      for (uint32_t i = 0; i < 3; ++i) {
        const uint32_t low = (rec[j].w >> (10 * i)) & 1023u;
        const bool in = i < rec[j].z;
        ta += in && low > b3;
        tt += in && low == b3;
      }
    }
  }
  if (__syncthreads_or(bad)) return;   // CTA-uniform: the write kernel's look-back takes the segment
  const uint2 ex = scan_excl2<NT>(ta, tt, sh);
  uint32_t ea = ex.x, et = ex.y;
  unsigned long long* lb = reinterpret_cast<unsigned long long*>(S.gcnt);
  for (uint32_t gb = g0; gb < g1; gb += kScanB) {
    uint4 rec[kScanB];
#pragma unroll
    for (int j = 0; j < kScanB; ++j) rec[j] = gb + j < g1 ? rec_of(gb + j) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < kScanB; ++j) {
      if (gb + j >= g1) break;
      lb[gb + j] = lb_pack(3, ea, et);
      ea += rec[j].y;
#pragma unroll
      for (uint32_t i = 0; i < 3; ++i) {
        const uint32_t low = (rec[j].w >> (10 * i)) & 1023u;
        const bool in = i < rec[j].z;
        ea += in && low > b3;
        et += in && low == b3;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 5) dgc_write_kernel(const SegH1* __restrict__ segs,
                                                             const uint32_t* __restrict__ group_seg,
                                                             uint32_t ngroups) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  __shared__ uint32_t sh_zc[kWarpsPerCta][kRunsPerGroup / 8];   // deferred zeroing: per tile of the group
  // ... and the group's records, assembled here and stored whole (full
  // sectors: no DRAM read-modify-write of partly written record lines)
  __shared__ __align__(16) uint16_t sh_zr[kWarpsPerCta][kRunsPerGroup / 8][kZRecMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t gi = blockIdx.x * kWarpsPerCta + w;
  if (gi < ngroups) {
    const WarpGroup G = warp_group_dense(segs, group_seg, gi);
    const SegH1& S = *G.S;
    const uint32_t C = G.C, g = G.g;
    const uint2* dense = group_slots(G);
    const uint32_t T = __ldcg(&S.st->prefix);
    const uint32_t need = __ldcg(&S.st->need);
    unsigned long long* lb = reinterpret_cast<unsigned long long*>(S.gcnt);
    const unsigned long long pre = __ldcg(lb + g);
    uint32_t ea = 0, et = 0;
    if ((uint32_t)(pre >> 62) == 3) {   // dgc_scan_kernel's exclusive prefix
      ea = (uint32_t)((pre >> 31) & 0x7FFFFFFFu);
      et = (uint32_t)(pre & 0x7FFFFFFFu);
    } else {
      // pass 1: the group's aggregate -- from refine<3>'s record when at most
      // three candidates fell into T's 21-bit bin (almost always), else counted
      uint32_t above = 0, tie = 0;
      const uint32_t* rec = S.runcnt + (size_t)g * S.rpg;
      const uint32_t r_in = __ldcg(rec + 2);
      if (r_in <= 3) {
        if (lane == 0) {
          const uint32_t b3 = T & 1023u, pk = __ldcg(rec + 3);
          above = __ldcg(rec + 1);
          for (uint32_t i = 0; i < r_in; ++i) {
            const uint32_t low = (pk >> (10 * i)) & 1023u;
            above += low > b3;
            tie += low == b3;
          }
        }
      } else
      for (uint32_t q0 = lane; q0 < C; q0 += kBatch * 32) {
        uint32_t key[kBatch];
#pragma unroll
        for (int m = 0; m < kBatch; ++m) {
          const uint32_t q = q0 + m * 32;
          key[m] = q < C ? __ldcg(&dense[q].y) & 0x7FFFFFFFu : 0u;
        }
#pragma unroll
        for (int m = 0; m < kBatch; ++m) {
          const bool in = q0 + m * 32 < C;
          above += in && key[m] > T;
          tie += in && key[m] == T;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        above += __shfl_xor_sync(0xffffffffu, above, o);
        tie += __shfl_xor_sync(0xffffffffu, tie, o);
      }
      // decoupled look-back over the segment's groups, 32 predecessors per step
      // (lane i reads group g-1-i of the window)
      if (lane == 0) atomicExch(&lb[g], lb_pack(g == 0 ? 2 : 1, above, tie));
      if (g > 0) {
        int top = (int)g - 1;
        while (true) {
          const int j = top - lane;
          unsigned long long v;
          if (j >= 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(lb + j) : "memory");
          else v = lb_pack(2, 0, 0);   // before the first group: an inclusive zero
          const uint32_t flag = (uint32_t)(v >> 62);
          if (__any_sync(0xffffffffu, flag == 0)) {
            __nanosleep(20);
            continue;   // a predecessor in the window has not published yet
          }
          const uint32_t inc = __ballot_sync(0xffffffffu, flag == 2);
          const int lim = inc ? __ffs(inc) - 1 : 31;   // nearest inclusive predecessor
          uint32_t a = lane <= lim ? (uint32_t)((v >> 31) & 0x7FFFFFFFu) : 0u;
          uint32_t t = lane <= lim ? (uint32_t)(v & 0x7FFFFFFFu) : 0u;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            t += __shfl_xor_sync(0xffffffffu, t, o);
          }
          ea += a;
          et += t;
          if (inc) break;
          top -= 32;
        }
        if (lane == 0) atomicExch(&lb[g], lb_pack(2, ea + above, et + tie));
      }
    }   // look-back path
    // pass 2: ordered selection; selected before this group = above_before + min(ties_before, need)
    uint32_t tie_run = et;
    uint32_t sel_run = ea + min(et, need);
    uint32_t* out_idx = reinterpret_cast<uint32_t*>(S.chunk);
    float* out_val = reinterpret_cast<float*>(S.chunk + 4 * (size_t)S.kpad);
    // deferred EF zeroing: the group's tiles (rpg / 8 of them) get records of
    // their selected offsets (slot = a per-tile shared counter; the order in a
    // record is immaterial), an overflowing record zeroes r / u directly
    uint32_t* wz = sh_zc[w];
    const uint32_t zt0 = g * (S.rpg / 8);
    if (S.zrec) {
      if (lane < kRunsPerGroup / 8) wz[lane] = 0u;
      __syncwarp();
    }
    // kBatch x 32 candidates in flight per step (large groups at 1% ratios)
    for (uint32_t q0 = 0; q0 < C; q0 += kBatch * 32) {
      uint2 cb[kBatch];
#pragma unroll
      for (int m = 0; m < kBatch; ++m) {
        const uint32_t q = q0 + m * 32 + lane;
        cb[m] = q < C ? __ldcg(dense + q) : make_uint2(0, 0);
      }
#pragma unroll
      for (int m = 0; m < kBatch; ++m) {
        if (q0 + m * 32 >= C) break;   // warp-uniform
        const uint2 c = cb[m];
        const uint32_t key = c.y & 0x7FFFFFFFu;
        const bool in = q0 + m * 32 + lane < C;
        const bool is_above = in && key > T, is_tie = in && key == T;
        const uint32_t tb = __ballot_sync(0xffffffffu, is_tie);
        const uint32_t trank = tie_run + __popc(tb & lt_mask);
        const bool sel = is_above || (is_tie && trank < need);
        const uint32_t sb = __ballot_sync(0xffffffffu, sel);
        const uint32_t pos = sel_run + __popc(sb & lt_mask);
        if (sel) {
          out_idx[pos] = c.x;
          out_val[pos] = __uint_as_float(c.y);
          const bool rec = S.zrec && !dgc_is_sample(S, c.x);
          const uint32_t slot = rec ? atomicAdd(&wz[(c.x >> 12) - zt0], 1u) : 0xFFFFFFFFu;
          if (rec && slot + 1 < S.zcap) {
            sh_zr[w][(c.x >> 12) - zt0][1 + slot] = (uint16_t)(c.x & (kDgcTile - 1));
          } else {   // no record, a full one, or a sample position: zeroed now
            if (S.ef) S.r[c.x] = 0.0f;
            if (S.mom) S.mom[c.x] = 0.0f;   // momentum factor masking (R20)
          }
        }
        tie_run += __popc(tb);
        sel_run += __popc(sb);
      }
    }
    if (S.zrec) {
      __syncwarp();
      const uint32_t ntiles = (S.n + kDgcTile - 1) / kDgcTile;
      const uint32_t nt = min(S.rpg / 8, ntiles - zt0);
      if ((uint32_t)lane < nt) sh_zr[w][lane][0] = (uint16_t)min(wz[lane], S.zcap - 1);
      __syncwarp();
      // the nt records (zcap uint16 each, contiguous in global memory) as 16-byte stores
      const uint32_t per = S.zcap / 8;   // uint4 per record
      uint4* dst = reinterpret_cast<uint4*>(S.zrec + (size_t)zt0 * S.zcap);
      for (uint32_t q = lane; q < nt * per; q += 32)
        dst[q] = *reinterpret_cast<const uint4*>(&sh_zr[w][q / per][(q % per) * 8]);
    }
    // approximate-count mode (R22): fewer than k entries may have been sent;
    // the segment's last group pads the rest of [0, k) (the chunk is reused)
    if (S.approx && g == S.ngroups - 1) {
      const uint32_t total = __ldcg(&S.st->above) + need;
      for (uint32_t q = total + lane; q < S.k; q += 32) {
        out_idx[q] = 0xFFFFFFFFu;
        out_val[q] = 0.0f;
      }
    }
  }
}

// Blocks the stream until *cnt >= target.  A peer that has not arrived after
// timeout_ns of wall time (%globaltimer, independent of the SM clock) is an
// error, not a hang: the kernel records it in the world's mapped error word
// and returns; esp_world_check and the next esp_sync* call report it (the
// consumers of this call then read an incomplete payload).  No __trap: a trap
// would destroy the CUDA context of the whole process.
// ------------------------------------------------------------------ small segments
// A bucket whose segments all have n <= kSample elements (one CTA per segment):
// the whole h1 -- acc = g + r (momentum: u = m u + g first), the exact k-th
// key by three radix rounds over the segment in shared memory, the ordered
// write and the EF update -- in ONE kernel instead of the sample / stream /
// fallback / refine / write chain, whose per-launch costs dominate at these
// sizes (P:1280's constant per-kernel overhead).  Same selection as the large
// pipeline: the top-k by (key desc, idx asc), emitted sorted by index.
__global__ void __launch_bounds__(kThreads) dgc_small_kernel(const SegH1* __restrict__ segs) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  __shared__ float acc[kSample];
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t sh[288];
  const SegH1& S = segs[blockIdx.x];
  const uint32_t n = S.n, k = S.k;
  const int tid = threadIdx.x;
  const float* g = seg_g(S);
  if (S.zrec) {   // a pending deferred zeroing (one tile): applied, r is rewritten below
    const uint32_t cnt = min((uint32_t)S.zrec[0], S.zcap - 1);
    for (uint32_t i = 1 + tid; i <= cnt; i += kThreads) {
      const uint32_t off = S.zrec[i];
      if (off < n) {
        if (S.ef) S.r[off] = 0.0f;
        if (S.mom) S.mom[off] = 0.0f;
      }
    }
    __syncthreads();
    if (tid == 0) S.zrec[0] = 0;
  }
  for (uint32_t i = tid; i < n; i += kThreads) {
    float x = __ldg(g + i);
    if (S.mom) {   // momentum correction (R20): u = fl(fl(m u) + g)
      x = __fadd_rn(__fmul_rn(S.mcoef, S.mom[i]), x);
      S.mom[i] = x;
    }
    acc[i] = S.ef ? __fadd_rn(x, S.r[i]) : x;
  }
  __syncthreads();
  // exact k-th key: 11 + 10 + 10 bits
  uint32_t prefix = 0, need = k, above = 0;
#pragma unroll 1
  for (int round = 1; round <= 3; ++round) {
    const int nb = round == 1 ? 2048 : 1024;
    const int shift_bin = round == 1 ? 20 : round == 2 ? 10 : 0;
    const int shift_match = round == 2 ? 20 : 10;
    for (int b = tid; b < nb; b += kThreads) hist[b] = 0;
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kThreads) {
      const uint32_t key = fkey(acc[i]);
      if (round == 1 || (key >> shift_match) == prefix) atomicAdd(&hist[(key >> shift_bin) & (nb - 1)], 1u);
    }
    __syncthreads();
    uint32_t bin, ab;
    select_bin<0, false>(hist, nb, need, &bin, &ab, sh);
    prefix = round == 1 ? bin : ((prefix << 10) | bin);
    above += ab;
    need -= ab;
  }
  const uint32_t T = prefix;
  // ordered write: a contiguous run of elements per thread
  const uint32_t per = (n + kThreads - 1) / kThreads;
  const uint32_t q0 = min(n, tid * per), q1 = min(n, q0 + per);
  uint32_t na = 0, nt = 0;
  for (uint32_t q = q0; q < q1; ++q) {
    const uint32_t key = fkey(acc[q]);
    na += key > T;
    nt += key == T;
  }
  uint32_t ta, tt;
  uint32_t ab = block_excl_scan<0>(na, &ta, sh);
  uint32_t tb = block_excl_scan<0>(nt, &tt, sh);
  uint32_t* out_idx = reinterpret_cast<uint32_t*>(S.chunk);
  float* out_val = reinterpret_cast<float*>(S.chunk + 4 * (size_t)S.kpad);
  for (uint32_t q = q0; q < q1; ++q) {
    const float a = acc[q];
    const uint32_t key = fkey(a);
    const bool is_above = key > T, is_tie = key == T;
    const bool sel = is_above || (is_tie && tb < need);
    if (sel) {
      const uint32_t pos = ab + min(tb, need);
      out_idx[pos] = q;
      out_val[pos] = a;
      if (S.mom) S.mom[q] = 0.0f;   // momentum factor masking (R20)
    }
    if (S.ef) S.r[q] = sel ? 0.0f : a;
    ab += is_above;
    tb += is_tie;
  }
}

// ------------------------------------------------------------------ on-chip h1
// DGC / TOPK h1 of a bucket that fits the chip's shared memory (every CTA holds
// <= kMidTpcMax tiles of acc = g + r): the whole h1 in ONE kernel instead of the
// seven-kernel chain, whose per-kernel latency is the cost at these sizes
// (BASELINE config 1 is a 2^20-element tensor).  Segment s gets
// ceil(tiles_s / tpc) CTAs of 1024 threads, all resident at once (grid <= #SMs,
// one CTA per SM by shared memory), which meet at four spin barriers on the
// segment's zeroed-every-call counters:
//   load    acc = g + r (u = m u + g first with momentum, R20) into shared
//           memory + the slice's 2048-bin histogram of the top 11 key bits
//   round 1 (barrier) bin of the k-th key from the summed histogram; a pass
//           histograms the next 10 bits of that bin's keys
//   round 2 (barrier) next bin; a pass histograms the low 10 bits of its keys
//   round 3 (barrier) T = the exact k-th key; warp ballots give the bitmaps
//           key > T and key == T (1 bit per element)
//   count   (barrier) every CTA's (#above T, #ties) -> the selected in the CTAs
//           before it and the ties it may take (ascending index); a CTA scan
//           of the bitmap words places each selected element in the
//           index-sorted payload; then r := acc with 0 where selected (a
//           float4 pass) and u := 0 there.
// No sampled threshold and no candidate list: the exact k-th key T and the
// (key desc, idx asc) selection are the same as the chain's (reading R3).
constexpr uint32_t kMidTpcMax = 12;   // 192 KB of acc (the bitmaps of 12 tiles fill the 3072 histogram words)
constexpr uint32_t kMidSmem = kMidTpcMax * kDgcTile * 4;

__device__ __forceinline__ void seg_barrier(uint32_t* ctr, uint32_t expected) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release: the CTA's writes before the bar.sync above are ordered before
    // the arrival (no full fence.sc)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    uint32_t v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= expected) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

constexpr int kMidThreads = 1024;   // 32 warps: the passes are latency-bound chains
constexpr int kMidWarps = kMidThreads / 32;

// exclusive scan of v over the 1024 threads in thread order; sh needs 33 words
__device__ __forceinline__ uint32_t mid_excl_scan(uint32_t v, uint32_t* total, uint32_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = sh[lane];
    uint32_t s2 = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s2, o);
      if (lane >= o) s2 += y;
    }
    sh[lane] = s2 - w;
    if (lane == 31) sh[32] = s2;
  }
  __syncthreads();
  const uint32_t r = x - v + sh[warp];
  *total = sh[32];
  __syncthreads();
  return r;
}

// CTA-wide radix bin choice by the first 256 threads (select_bin on named
// barrier 1), broadcast through shared memory; GLOBAL: the segment's summed
// histogram in global memory, else this CTA's own (a one-CTA segment)
template <bool GLOBAL = true>
__device__ __forceinline__ uint2 mid_select(const uint32_t* gh, int nbins, uint32_t need, uint32_t* sh,
                                            uint32_t* res) {
  if (threadIdx.x < kThreads) {
    uint32_t b, a;
    select_bin<1, GLOBAL>(gh, nbins, need, &b, &a, sh);
    if (threadIdx.x == 0) {
      res[0] = b;
      res[1] = a;
    }
  }
  __syncthreads();
  return make_uint2(res[0], res[1]);
}

__global__ void __launch_bounds__(kMidThreads, 1) dgc_mid_kernel(const SegH1* __restrict__ segs, int nsegs,
                                                                 uint32_t tpc) {
  extern __shared__ float4 mid_smem4[];
  float* acc = reinterpret_cast<float*>(mid_smem4);
  __shared__ uint32_t hist12[3072];   // round 1 (2048 bins) + rounds 2 / 3 (1024); then the bitmaps
  uint32_t* hist1 = hist12;
  uint32_t* hist2 = hist12 + 2048;
  __shared__ uint32_t sh[288];
  __shared__ uint32_t info[6];   // segment, CTA index in it, CTAs of it, (unused), select result (2)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // CTA -> (segment, index) from the static table (before pdl_wait)
  if (tid < kThreads) {
    const uint32_t c = tid < nsegs ? ((segs[tid].n + kDgcTile - 1) / kDgcTile + tpc - 1) / tpc : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<1>(c, &tot, sh);
    if (c && blockIdx.x >= ex && blockIdx.x < ex + c) {
      info[0] = tid;
      info[1] = blockIdx.x - ex;
      info[2] = c;
    }
  }
  for (int b = tid; b < 2048; b += kMidThreads) hist1[b] = 0;
  for (int b = tid; b < 1024; b += kMidThreads) hist2[b] = 0;
  __syncthreads();
  const SegH1& S = segs[info[0]];
  const uint32_t ci = info[1], nc = info[2];
  const uint32_t n = S.n, k = S.k;
  const uint32_t lo = ci * tpc * kDgcTile, hi = min(n, lo + tpc * kDgcTile), len = hi - lo;
  pdl_wait();
  pdl_trigger();
  const bool ef = S.ef != 0;
  float* r = ef ? S.r + lo : nullptr;
  float* u = S.mom ? S.mom + lo : nullptr;
  const float m = S.mcoef;
  const float* g = seg_g(S) + lo;
  if (S.zrec) {   // pending deferred zeroing of this CTA's tiles (a chained call before): applied first
    const uint32_t t0 = lo / kDgcTile, t1 = (hi + kDgcTile - 1) / kDgcTile;
    for (uint32_t t = t0 + warp; t < t1; t += kMidWarps) {
      uint16_t* z = S.zrec + (size_t)t * S.zcap;
      const uint32_t cnt = min((uint32_t)z[0], S.zcap - 1);
      for (uint32_t i = 1 + lane; i <= cnt; i += 32) {
        const uint32_t e = t * kDgcTile + z[i];
        if (e < n) {
          if (ef) S.r[e] = 0.0f;
          if (S.mom) S.mom[e] = 0.0f;
        }
      }
      __syncwarp();
      if (lane == 0) z[0] = 0;
    }
    __syncthreads();
  }
  // ---- load: acc = g + r, histogram of the top 11 key bits (atomicAdd(.., 1)
  // compiles to ATOMS.POPC.INC: the lanes of a warp that hit one bin are one update)
  auto elem = [&](float x, float rv, float uv, float& uo) {
    uo = 0.0f;
    if (u) {   // momentum correction (R20): u = fl(fl(m u) + g)
      x = __fadd_rn(__fmul_rn(m, uv), x);
      uo = x;
    }
    return ef ? __fadd_rn(x, rv) : x;
  };
  const bool vec = al16(g) && (!ef || al16(r)) && (!u || al16(u));
  const uint32_t n4 = vec ? len / 4 : 0;
  // batches of kB float4 per thread, every load of a batch issued before any use
  // (~64 KB in flight per SM: one CTA per SM has to cover the DRAM latency alone)
  constexpr int kB = 2;
  for (uint32_t i0 = 0; i0 < n4; i0 += kB * kMidThreads) {
    float4 x[kB], rv[kB], uv[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const uint32_t i = i0 + j * kMidThreads + tid;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      x[j] = i < n4 ? ld_stream4(g + 4 * i) : z;
      rv[j] = ef && i < n4 ? ld4(r + 4 * i) : z;
      uv[j] = u && i < n4 ? ld4(u + 4 * i) : z;
    }
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const uint32_t i = i0 + j * kMidThreads + tid;
      const bool v = i < n4;
      float4 a, uo;
      a.x = elem(x[j].x, rv[j].x, uv[j].x, uo.x);
      a.y = elem(x[j].y, rv[j].y, uv[j].y, uo.y);
      a.z = elem(x[j].z, rv[j].z, uv[j].z, uo.z);
      a.w = elem(x[j].w, rv[j].w, uv[j].w, uo.w);
      if (v) {
        if (u) st4(u + 4 * i, uo);
        *reinterpret_cast<float4*>(acc + 4 * i) = a;
      }
      if (v) atomicAdd(&hist1[fkey(a.x) >> 20], 1u);
      if (v) atomicAdd(&hist1[fkey(a.y) >> 20], 1u);
      if (v) atomicAdd(&hist1[fkey(a.z) >> 20], 1u);
      if (v) atomicAdd(&hist1[fkey(a.w) >> 20], 1u);
    }
  }
  for (uint32_t i0 = 4 * n4; i0 < len; i0 += kMidThreads) {   // unaligned slices and the tail
    const uint32_t i = i0 + tid;
    if (i < len) {
      float uo;
      const float a = elem(g[i], ef ? r[i] : 0.0f, u ? u[i] : 0.0f, uo);
      if (u) u[i] = uo;
      acc[i] = a;
      atomicAdd(&hist1[fkey(a) >> 20], 1u);
    }
  }
  __syncthreads();
  // a one-CTA segment selects from its own shared histograms: no flush, no barrier
  const bool solo = nc == 1;
  if (!solo) {
    for (int b = tid; b < 2048; b += kMidThreads)
      if (hist1[b]) atomicAdd(S.hist + b, hist1[b]);
    seg_barrier(&S.st->done, nc);
  }
  // after round 3 the histogram words hold the bitmaps, 1 bit per element of
  // the slice (<= 12 tiles: 1536 words each)
  uint32_t* selbits = hist12;          // key > T (then: selected)
  uint32_t* tiebits = hist12 + 1536;   // key == T
  uint2 sel = solo ? mid_select<false>(hist1, 2048, k, sh, info + 4)
                   : mid_select(S.hist, 2048, k, sh, info + 4);   // (its __syncthreads orders the flush reads)
  const uint32_t bin1 = sel.x;
  uint32_t need = k - sel.y;
  // ---- round 2: the next 10 key bits of round 1's bin (a float4 per thread)
  for (uint32_t i = 4 * tid; i < len; i += 4 * kMidThreads) {
    const float4 a4 = lds4(acc + i);   // (beyond len: stale shared memory, masked below)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t key = fkey(f4get(a4, c));
      if (i + c < len && (key >> 20) == bin1) atomicAdd(&hist2[(key >> 10) & 1023], 1u);
    }
  }
  __syncthreads();
  uint32_t* gh2 = S.hist + 4096;
  uint32_t* gh3 = S.hist + 4096 + 1024 * S.hrep;
  if (solo) {
    sel = mid_select<false>(hist2, 1024, need, sh, info + 4);
    for (int b = tid; b < 1024; b += kMidThreads) hist2[b] = 0;   // reused by round 3
    __syncthreads();
  } else {
    for (int b = tid; b < 1024; b += kMidThreads) {
      if (hist2[b]) atomicAdd(gh2 + b, hist2[b]);
      hist2[b] = 0;   // reused by round 3 (the barrier below orders it)
    }
    seg_barrier(&S.st->done_r2, nc);
    sel = mid_select(gh2, 1024, need, sh, info + 4);
  }
  const uint32_t prefix2 = (bin1 << 10) | sel.x;
  need -= sel.y;
  // ---- round 3: the low 10 bits of the keys in round 2's bin
  for (uint32_t i = 4 * tid; i < len; i += 4 * kMidThreads) {
    const float4 a4 = lds4(acc + i);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t key = fkey(f4get(a4, c));
      if (i + c < len && (key >> 10) == prefix2) atomicAdd(&hist2[key & 1023], 1u);
    }
  }
  __syncthreads();
  if (solo) {
    sel = mid_select<false>(hist2, 1024, need, sh, info + 4);
  } else {
    for (int b = tid; b < 1024; b += kMidThreads)
      if (hist2[b]) atomicAdd(gh3 + b, hist2[b]);
    seg_barrier(&S.st->done_r3, nc);
    sel = mid_select(gh3, 1024, need, sh, info + 4);
  }
  const uint32_t T = (prefix2 << 10) | sel.x;
  need -= sel.y;   // the ties at T to take, by ascending index
  // ---- bitmaps by warp ballots over 32 consecutive elements: key > T, key == T
  const uint32_t nwords = (len + 31) / 32;
  for (uint32_t w = warp; w < nwords; w += kMidWarps) {
    const uint32_t i = w * 32 + lane;
    const uint32_t key = i < len ? fkey(acc[i]) : 0u;
    const unsigned ma = __ballot_sync(0xffffffffu, i < len && key > T);
    const unsigned mt = __ballot_sync(0xffffffffu, i < len && key == T);
    if (lane == 0) {
      selbits[w] = ma;
      tiebits[w] = mt;
    }
  }
  __syncthreads();
  // thread t owns words 2t and 2t + 1 (elements 64t .. 64t + 63) from here on
  const uint32_t w0 = 2 * tid;
  uint32_t s0 = w0 < nwords ? selbits[w0] : 0u, s1 = w0 + 1 < nwords ? selbits[w0 + 1] : 0u;
  const uint32_t t0 = w0 < nwords ? tiebits[w0] : 0u, t1 = w0 + 1 < nwords ? tiebits[w0 + 1] : 0u;
  // ---- count: (#above T, #ties) of this CTA, published; the CTAs before it
  uint32_t ca = __popc(s0) + __popc(s1), ct = __popc(t0) + __popc(t1);
  const uint2 ex = scan_excl2<kMidThreads>(ca, ct, sh);   // within the CTA, in element order
  uint2* slots = S.cand;   // per CTA: (#above T, #ties) (the chain's candidate buffer)
  if (!solo) {
    if (tid == kMidThreads - 1) {
      const uint32_t ta = ex.x + ca, tt = ex.y + ct;
      __stcg(reinterpret_cast<unsigned long long*>(slots + ci), ((unsigned long long)tt << 32) | ta);
    }
    seg_barrier(&S.st->done_cnt, nc);
  }
  if (warp == 0) {
    uint32_t ba = 0, bt = 0;
    for (uint32_t j = lane; j < ci; j += 32) {
      const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long*>(slots + j));
      ba += (uint32_t)v;
      bt += (uint32_t)(v >> 32);
    }
    ba = __reduce_add_sync(0xffffffffu, ba);
    bt = __reduce_add_sync(0xffffffffu, bt);
    if (lane == 0) {
      info[4] = ba;
      info[5] = bt;
    }
  }
  __syncthreads();
  const uint32_t cabove = info[4], ctie = info[5];
  // ties by ascending index: a tie with tbase ties before it is taken iff tbase < need
  {
    uint32_t tb = ctie + ex.y;
    for (int h = 0; h < 2; ++h) {
      uint32_t tw = h ? t1 : t0;
      while (tw) {
        const uint32_t bit = __ffs(tw) - 1;
        tw &= tw - 1;
        if (tb < need) (h ? s1 : s0) |= 1u << bit;
        ++tb;
      }
    }
  }
  // selected before this pair: above in the CTAs before + the ties they took +
  // this CTA's selected before the pair (scan of the final words)
  const uint2 ex2 = scan_excl2<kMidThreads>(__popc(s0) + __popc(s1), 0u, sh);
  const uint32_t cbase = cabove + min(ctie, need) + ex2.x;
  if (w0 < nwords) selbits[w0] = s0;
  if (w0 + 1 < nwords) selbits[w0 + 1] = s1;
  // ---- ordered write: idx / val of the selected, u := 0 there
  uint32_t* out_idx = reinterpret_cast<uint32_t*>(S.chunk);
  float* out_val = reinterpret_cast<float*>(S.chunk + 4 * (size_t)S.kpad);
  {
    uint32_t pos = cbase;
    for (int h = 0; h < 2; ++h) {
      uint32_t sw = h ? s1 : s0;
      while (sw) {
        const uint32_t e = (w0 + h) * 32 + __ffs(sw) - 1;
        sw &= sw - 1;
        out_idx[pos] = lo + e;
        out_val[pos] = acc[e];
        if (u) u[e] = 0.0f;   // momentum factor masking (R20)
        ++pos;
      }
    }
  }
  __syncthreads();   // the final selbits
  // ---- r := acc, 0 where selected (a float4 per thread and step)
  if (ef) {
    const bool rvec = al16(r);
    for (uint32_t i = 4 * tid; i < len; i += 4 * kMidThreads) {
      float4 a4 = lds4(acc + i);
      const uint32_t sb = selbits[i >> 5] >> (i & 31);
      if (sb & 1u) a4.x = 0.0f;
      if (sb & 2u) a4.y = 0.0f;
      if (sb & 4u) a4.z = 0.0f;
      if (sb & 8u) a4.w = 0.0f;
      if (rvec && i + 3 < len) {
        st4(r + i, a4);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (i + c < len) r[i + c] = f4get(a4, c);
      }
    }
  }
}

// Applies a segment's pending deferred zeroing to r and u in memory and clears
// the records (state read-out: esp_ctx_get_state / get_momentum).  One warp
// per tile.
__global__ void dgc_zrec_apply_kernel(float* r, float* u, uint16_t* zrec, uint32_t zcap, uint32_t n) {
  const uint32_t t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= (n + kDgcTile - 1) / kDgcTile) return;
  uint16_t* z = zrec + (size_t)t * zcap;
  const uint32_t cnt = min((uint32_t)z[0], zcap - 1);
  for (uint32_t i = 1 + lane; i <= cnt; i += 32) {
    const uint32_t e = t * kDgcTile + z[i];
    if (e < n) {
      if (r) r[e] = 0.0f;
      if (u) u[e] = 0.0f;
    }
  }
  __syncwarp();
  if (lane == 0) z[0] = 0;
}

void launch_dgc_zrec_apply(float* r, float* u, uint16_t* zrec, uint32_t zcap, uint32_t n, cudaStream_t st) {
  if (!zrec || n == 0) return;
  const uint32_t ntiles = (n + kDgcTile - 1) / kDgcTile;
  dgc_zrec_apply_kernel<<<(ntiles + 7) / 8, 256, 0, st>>>(r, u, zrec, zcap, n);
  count_launches(1);
}

uint32_t dgc_mid_tpc_max() { return kMidTpcMax; }

void launch_dgc_mid(const SegH1* segs, int nsegs, uint32_t tpc, int grid, cudaStream_t st) {
  if (nsegs == 0 || grid == 0) return;
  static const bool attr_set =
      cudaFuncSetAttribute(dgc_mid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMidSmem) ==
      cudaSuccess;
  (void)attr_set;
  launch_pdl(dgc_mid_kernel, grid, kMidThreads, (size_t)tpc * kDgcTile * 4, st, segs, nsegs, tpc);
  count_launches(1);
}

void launch_dgc_small(const SegH1* segs, int nsegs, cudaStream_t st) {
  if (nsegs == 0) return;
  launch_pdl(dgc_small_kernel, nsegs, kThreads, 0, st, segs);
  count_launches(1);
}

__global__ void wait_arrivals_kernel(const unsigned long long* cnt, unsigned long long target,
                                     unsigned int* err, unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t sleep = 32;
  while (true) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
    if (v >= target) break;
    __nanosleep(sleep);
    if (sleep < 1024) sleep <<= 1;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicExch_system(err, 1u);
      __threadfence_system();
      break;
    }
  }
}

void launch_wait_arrivals(const unsigned long long* cnt, unsigned long long target, unsigned int* err,
                          unsigned long long timeout_ns, cudaStream_t st) {
  if (target == 0) return;   // nothing to wait for (e.g. the root's own broadcast)
  wait_arrivals_kernel<<<1, 32, 0, st>>>(cnt, target, err, timeout_ns);
  count_launches(1);
}

// ------------------------------------------------------------------ launchers
static int g_num_sms = 0;

static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

// persistent streaming kernels: one CTA per SM (measured best on B200)
int tma_stream_grid(int nunits) { return nunits < num_sms() ? nunits : num_sms(); }

// ring depth of the streaming kernels (measured flat from 3 to 6 on B200)
int tma_stream_stages() { return 4; }

// ESP_DEBUG_SYNC=1: synchronize after every kernel of the DGC pipeline and name
// the one that failed (debugging aid; off by default)
static void debug_sync(const char* what, cudaStream_t st) {
  static const bool on = [] {
    const char* e = getenv("ESP_DEBUG_SYNC");
    return e && atoi(e) != 0;
  }();
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    fprintf(stderr, "[esp] %s failed: %s\n", what, cudaGetErrorString(e));
    fflush(stderr);
  }
}

void launch_dgc_h1(const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits,
                   const uint32_t* group_seg, int ngroups, cudaStream_t st, cudaEvent_t probe0,
                   cudaEvent_t probe1, bool mom) {
  launch_dgc_stream(segs, nsegs, unit_seg, nunits, st, probe0, probe1, mom);
  launch_dgc_finalize(segs, nsegs, group_seg, ngroups, st);
}

void launch_dgc_stream(const SegH1* segs, int nsegs, const uint32_t* unit_seg, int nunits, cudaStream_t st,
                       cudaEvent_t probe0, cudaEvent_t probe1, bool mom) {
  if (nsegs == 0) return;
  // three consumer groups of 8 warps over a 3-stage ring of 32 KB (plain EF);
  // two groups over 4 stages of 48 KB with the momentum stream (R20) -- the
  // configurations measured fastest on B200 (DESIGN.md tuning log)
  constexpr int kNs = 3, kNsMom = 4;
  const size_t smem = kStreamHdr + kNs * kStageBytes;
  const size_t mom_smem = kStreamHdr + kNsMom * kStageBytesMom;
  static const bool attr_set = [&] {
    return cudaFuncSetAttribute(dgc_stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
               cudaSuccess &&
           cudaFuncSetAttribute(dgc_stream_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)mom_smem) == cudaSuccess;
  }();
  (void)attr_set;
  num_sms();
  const char* ff = getenv("ESP_DGC_FORCE_FALLBACK");   // read per launch: a test hook
  // sample-rank margin in standard deviations of the sample count (4: 2 and 1
  // measured to send segments through the fallback recompaction)
  constexpr float kMargin = 4.0f;
  launch_pdl(dgc_sample_kernel, nsegs, kThreads, 0, st, segs, ff ? atoi(ff) : 0, kMargin);
  debug_sync("dgc_sample", st);
  if (probe0) cudaEventRecord(probe0, st);
  const int grid = nunits < g_num_sms ? nunits : g_num_sms;
  if (mom)
    launch_pdl(dgc_stream_kernel<2, true>, grid, 2 * kThreads + 32, mom_smem, st, segs, unit_seg, (uint32_t)nunits,
               kNsMom);
  else
    launch_pdl(dgc_stream_kernel<3>, grid, 3 * kThreads + 32, smem, st, segs, unit_seg, (uint32_t)nunits, kNs);
  debug_sync("dgc_stream", st);
  if (probe1) cudaEventRecord(probe1, st);
  count_launches(2);
}

void launch_dgc_finalize(const SegH1* segs, int nsegs, const uint32_t* group_seg, int ngroups, cudaStream_t st) {
  if (nsegs == 0) return;
  num_sms();
  launch_pdl(dgc_fallback_kernel, g_num_sms, kThreads, 0, st, segs, nsegs);
  debug_sync("dgc_fallback", st);
  const int wgrid = (ngroups + kWarpsPerCta - 1) / kWarpsPerCta;   // one warp per finalize group
  // many groups per segment (1% ratios on large tensors): selects as kernels
  const bool sep = ngroups > kSepGroupsPerSeg * nsegs;
  if (wgrid > 0) {
    if (sep) {
      launch_pdl(dgc_refine_kernel<2, false>, wgrid, kThreads, 0, st, segs, group_seg, (uint32_t)ngroups);
      launch_pdl(dgc_select_kernel<2>, nsegs, 32, 0, st, segs);
      launch_pdl(dgc_refine_kernel<3, false>, wgrid, kThreads, 0, st, segs, group_seg, (uint32_t)ngroups);
      launch_pdl(dgc_select_kernel<3>, nsegs, 32, 0, st, segs);
    } else {
      launch_pdl(dgc_refine_kernel<2, true>, wgrid, kThreads, 0, st, segs, group_seg, (uint32_t)ngroups);
      debug_sync("dgc_refine<2>", st);
      launch_pdl(dgc_refine_kernel<3, true>, wgrid, kThreads, 0, st, segs, group_seg, (uint32_t)ngroups);
    }
    debug_sync("dgc_refine<3>", st);
    if (ngroups > 2048 * nsegs)
      launch_pdl(dgc_scan_kernel<1024>, nsegs, 1024, 0, st, segs);
    else
      launch_pdl(dgc_scan_kernel<256>, nsegs, 256, 0, st, segs);
    launch_pdl(dgc_write_kernel, wgrid, kThreads, 0, st, segs, group_seg, (uint32_t)ngroups);
    debug_sync("dgc_write", st);
  }
  count_launches(wgrid > 0 ? (sep ? 7 : 5) : 1);
}

}  // namespace esp
