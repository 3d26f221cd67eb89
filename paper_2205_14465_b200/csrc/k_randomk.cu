// Randomk on sm_100a (Randomk evaluated at a 1% rate,
// P:1426; EF at P:1427).
//
// h1: one fused pass (12 B/elem) on the persistent TMA streaming driver: acc =
// g + r; each stratum j = [floor(jN/k), floor((j+1)N/k)) picks one element
// (reading R5); val[j] = acc[pick]; r := picked ? 0 : acc.  The work is
// organised per stratum, not per element: a warp's 512-element run meets only
// ~ρ·512 strata, whose picks (one 64-bit hash and division each) are computed
// one per lane and applied through a per-warp shared-memory copy of the run's
// acc values and a 512-bit pick mask.
//
// h2: per 8192-element tile, the picks of the tile's strata are accumulated
// in shared memory piece by piece in rank order (every piece touches distinct
// positions), then the tile is written once (÷ n).
#include "esp_device.cuh"
#include "esp_kernels.h"
#include "stream_tma.cuh"

namespace esp {

__device__ __forceinline__ uint64_t stratum_of(uint64_t i, uint64_t k, uint64_t n) {
  return ((i + 1) * k + n - 1) / n - 1;
}

// The oracle's chain (reading R5): h = mix(mix(mix(mix(mix(seed)^tensor)^step)^part)^rankterm),
// pick_j = start_j + mix(h ^ j) mod len_j.  `base` = mix(mix(seed)^tensor) from the planner.
__device__ __forceinline__ uint64_t randomk_hash(uint64_t base, uint64_t step, uint32_t part,
                                                  uint32_t rankterm) {
  return splitmix64(splitmix64(splitmix64(base ^ step) ^ (uint64_t)part) ^ (uint64_t)rankterm);
}

__device__ __forceinline__ uint32_t randomk_pick(uint64_t h, uint64_t j, uint64_t k, uint64_t n) {
  const uint64_t a = j * n / k, b = (j + 1) * n / k;
  return (uint32_t)(a + splitmix64(h ^ j) % (b - a));
}

// ------------------------------------------------------------------ h1
struct RandomkOp {
  static constexpr int kGroups = 3;   // consumer groups
  struct State {
    uint64_t h;
  };
  const unsigned char* const* pieces = nullptr;   // not a decoding op
  bool stage_words = false;
  template <int BAR>
  __device__ void begin_segment(const SegH1& S, State& st, TmaGroup&) const {
    st.h = randomk_hash(S.hash, *S.step, S.part, S.rankterm);
  }
  template <bool FULL>
  __device__ void run(const SegH1& S, const float4 (&gv)[kNJ], const float4 (&rv)[kNJ], uint32_t base,
                      State& st, TmaGroup& hd, const uint32_t*) const {
    const uint32_t n = S.n, k = S.k;
    if (base >= n) return;   // warp-uniform
    const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 7;   // warp within the group
    float* scr = hd.wscr[warp];
    uint32_t* msk = hd.wsel[warp];
    float4 av[kNJ];
#pragma unroll
    for (int j = 0; j < kNJ; ++j) {
      av[j] = gv[j];
      if (S.ef) {
        av[j].x = __fadd_rn(gv[j].x, rv[j].x);
        av[j].y = __fadd_rn(gv[j].y, rv[j].y);
        av[j].z = __fadd_rn(gv[j].z, rv[j].z);
        av[j].w = __fadd_rn(gv[j].w, rv[j].w);
      }
      *reinterpret_cast<float4*>(scr + j * 128 + lane * 4) = av[j];
    }
    if (lane < kRun / 32) msk[lane] = 0u;
    __syncwarp();
    const uint32_t hi = min(base + (uint32_t)kRun, n) - 1;   // last element of the run
    const uint64_t j0 = stratum_of(base, k, n), j1 = stratum_of(hi, k, n);
    float* val = reinterpret_cast<float*>(S.chunk);
    for (uint64_t jb = j0; jb <= j1; jb += 32) {
      const uint64_t jj = jb + lane;
      if (jj <= j1) {
        const uint32_t p = randomk_pick(st.h, jj, k, n);
        if (p >= base && p <= hi) {   // the boundary strata may pick outside the run
          const uint32_t off = p - base;
          val[jj] = scr[off];
          atomicOr(&msk[off >> 5], 1u << (off & 31));
        }
      }
    }
    __syncwarp();
    if (!S.ef) return;
#pragma unroll
    for (int j = 0; j < kNJ; ++j) {
      const uint32_t off = j * 128 + lane * 4;
      const uint32_t sel = (msk[off >> 5] >> (off & 31)) & 0xFu;
      float4 nr = av[j];
      if (sel & 1) nr.x = 0.f;
      if (sel & 2) nr.y = 0.f;
      if (sel & 4) nr.z = 0.f;
      if (sel & 8) nr.w = 0.f;
      if (FULL) st4(S.r + base + off, nr);
      else store4_guard(S.r, base + off, n, nr);
    }
  }
  template <int BAR>
  __device__ void end_segment(const SegH1&, uint32_t, uint32_t, State&, TmaGroup&) const {}
};

// ------------------------------------------------------------------ h2
// out = reduce(sum over pieces of the scattered values); each piece carries
// its own hash (identical for all pieces when indices are shared).  Strata are
// disjoint ranges, so every output position can only be picked by ONE stratum
// (whatever the piece): one thread per stratum owns its positions and sums the
// pieces' values there in rank order from +0 -- no barrier between pieces.
// The stratum bounds are computed once, the pick once when every piece shares
// the indices (else one per piece, independent, so they overlap), and all of
// a batch's value loads are in flight before the first is added.
constexpr int kRkBatch = 8;
// Persistent: a few CTAs per SM, each over a contiguous range of the bucket's
// units, the segment prologue (piece hashes and pointers) once per (CTA,
// segment); per unit the 32 KB output tile is built in shared memory and
// stored once, while the next unit's picks are already being computed.
__global__ void __launch_bounds__(kThreads) h2_randomk_kernel(const SegH2* __restrict__ segs,
                                                              const uint32_t* __restrict__ unit_seg,
                                                              uint32_t nunits,
                                                              const unsigned char* const* __restrict__ pieces,
                                                              const uint32_t* __restrict__ rankterms) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  __shared__ __align__(16) float acc[kUnit];
  __shared__ uint64_t sh_h[64];
  __shared__ const float* sh_v[64];
  __shared__ int sh_shared;
  const uint32_t u0 = (uint32_t)((uint64_t)blockIdx.x * nunits / gridDim.x);
  const uint32_t u1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * nunits / gridDim.x);
  uint32_t cur = 0xFFFFFFFFu;
  SegH2 S{};
  bool shared = true;
  for (uint32_t gu = u0; gu < u1; ++gu) {
    const uint32_t sid = unit_seg[gu];
    __syncthreads();   // the previous unit's tile has been stored (and its segment's tables read)
    if (sid != cur) {
      cur = sid;
      S = segs[sid];
      const uint64_t step = *S.step;
      for (uint32_t r = threadIdx.x; r < S.npieces; r += kThreads) {
        sh_h[r] = randomk_hash(S.hash, step, S.part, rankterms[S.piece0 + r]);
        sh_v[r] = reinterpret_cast<const float*>(pieces[S.piece0 + r]);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int same = 1;
        for (uint32_t r = 1; r < S.npieces; ++r) same &= sh_h[r] == sh_h[0];
        sh_shared = same;
      }
    }
    for (int i = threadIdx.x; i < kUnit / 4; i += kThreads)
      reinterpret_cast<float4*>(acc)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    shared = sh_shared != 0;
    const uint32_t n = S.n, k = S.k, np = S.npieces;
    const uint32_t u = gu - S.unit0;
    const uint32_t lo = u * kUnit, hi = min(lo + (uint32_t)kUnit, n) - 1;
    const uint64_t j0 = stratum_of(lo, k, n), j1 = stratum_of(hi, k, n);
    for (uint64_t jj = j0 + threadIdx.x; jj <= j1; jj += kThreads) {
      const uint64_t a = jj * n / k, len = (jj + 1) * n / k - a;
      const uint32_t p0 = (uint32_t)(a + splitmix64(sh_h[0] ^ jj) % len);
      float sum = 0.f;
      bool any = false;
      uint32_t pos = 0;
      for (uint32_t r0 = 0; r0 < np; r0 += kRkBatch) {
        uint32_t p[kRkBatch];
        float v[kRkBatch];
#pragma unroll
        for (int m = 0; m < kRkBatch; ++m) {
          const uint32_t r = r0 + m;
          p[m] = (r < np) ? (shared || r == 0 ? p0 : (uint32_t)(a + splitmix64(sh_h[r] ^ jj) % len)) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int m = 0; m < kRkBatch; ++m) {
          const uint32_t r = r0 + m;
          v[m] = (r < np && p[m] >= lo && p[m] <= hi) ? __ldg(sh_v[r] + jj) : 0.f;
        }
#pragma unroll
        for (int m = 0; m < kRkBatch; ++m) {
          const uint32_t r = r0 + m;
          if (r < np && p[m] >= lo && p[m] <= hi) {
            if (shared) {
              sum = __fadd_rn(sum, v[m]);
              any = true;
              pos = p[m] - lo;
            } else {
              acc[p[m] - lo] = __fadd_rn(acc[p[m] - lo], v[m]);   // this thread owns the stratum's positions
            }
          }
        }
      }
      if (shared && any) acc[pos] = sum;
    }
    __syncthreads();
    const Divisor div(S.divisor);
    const bool ones = S.divisor == 1.0f;
    float* out = seg_out(S);
    for (uint32_t i = threadIdx.x * 4; lo + i <= hi; i += kThreads * 4) {
      float4 v = *reinterpret_cast<const float4*>(acc + i);
      if (!ones && (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f)) v = div(v);
      store4_guard(out, lo + i, n, v);
    }
  }
}

void launch_randomk_h1(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st) {
  if (nunits == 0) return;
  launch_tma_op(segs, unit_seg, nunits, RandomkOp{}, st);
}

void launch_h2_randomk(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                       const unsigned char* const* pieces, const uint32_t* rankterms, cudaStream_t st) {
  if (nunits == 0) return;
  static const int cap = [] {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2_randomk_kernel, kThreads, 0);
    return sms * (per_sm > 0 ? per_sm : 4);
  }();
  const int grid = nunits < cap ? nunits : cap;
  launch_pdl(h2_randomk_kernel, grid, kThreads, 0, st, segs, unit_seg, (uint32_t)nunits, pieces, rankterms);
  count_launches(1);
}

}  // namespace esp
