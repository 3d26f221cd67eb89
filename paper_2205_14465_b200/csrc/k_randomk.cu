// Randomk h1 on sm_100a (Randomk evaluated at a 1% rate,
// P:1426; EF at P:1427).  One fused pass (12 B/elem): acc = g + r; the element
// is selected iff it is the hashed pick of its stratum (reading R5); selected
// values go to val[j], and r := selected ? 0 : acc.
//
// Stratum j covers [floor(jN/k), floor((j+1)N/k)); element i lies in stratum
// ceil((i+1)k/N) - 1, so each float4 touches at most a few strata and needs
// one or two hashes instead of four.
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

__global__ void __launch_bounds__(kThreads) randomk_h1_kernel(const SegH1* __restrict__ segs,
                                                              const uint32_t* __restrict__ unit_seg) {
  const uint32_t sid = unit_seg[blockIdx.x];
  const SegH1 S = segs[sid];
  const uint32_t u = blockIdx.x - S.unit0;
  const uint32_t n = S.n, k = S.k;
  float* val = reinterpret_cast<float*>(S.chunk);
  const float* g = seg_g(S);
  const uint64_t h = randomk_hash(S.hash, *S.step, S.part, S.rankterm);
#pragma unroll 2
  for (int j = 0; j < kUnit / (kThreads * 4); ++j) {
    const uint32_t e = u * kUnit + (j * kThreads + threadIdx.x) * 4;
    if (e >= n) break;
    float4 acc = load4_stream_guard(g, e, n);
    if (S.ef) {
      const float4 r = load4_guard(S.r, e, n);
      acc.x = __fadd_rn(acc.x, r.x);
      acc.y = __fadd_rn(acc.y, r.y);
      acc.z = __fadd_rn(acc.z, r.z);
      acc.w = __fadd_rn(acc.w, r.w);
    }
    const uint32_t last = min(e + 3, n - 1);
    const uint64_t j0 = stratum_of(e, k, n), j1 = stratum_of(last, k, n);
    uint32_t sel = 0;
    for (uint64_t jj = j0; jj <= j1; ++jj) {
      const uint32_t idx = randomk_pick(h, jj, k, n);
      if (idx >= e && idx <= last) {
        sel |= 1u << (idx - e);
        val[jj] = f4get(acc, idx - e);
      }
    }
    if (S.ef) {
      float4 nr = acc;
      if (sel & 1) nr.x = 0.f;
      if (sel & 2) nr.y = 0.f;
      if (sel & 4) nr.z = 0.f;
      if (sel & 8) nr.w = 0.f;
      store4_guard(S.r, e, n, nr);
    }
  }
}

// h2 for Randomk: out = reduce(sum over pieces of the scattered values).  Each
// piece r carries its own hash base (identical for all r when indices are
// shared); contributions are added in rank order.
__global__ void __launch_bounds__(kThreads) h2_randomk_kernel(const SegH2* __restrict__ segs,
                                                              const uint32_t* __restrict__ unit_seg,
                                                              const unsigned char* const* __restrict__ pieces,
                                                              const uint32_t* __restrict__ rankterms) {
  const uint32_t sid = unit_seg[blockIdx.x];
  const SegH2 S = segs[sid];
  const uint32_t u = blockIdx.x - S.unit0;
  const uint32_t n = S.n, k = S.k;
  __shared__ uint64_t sh_h[64];
  const uint64_t step = *S.step;
  for (uint32_t r = threadIdx.x; r < S.npieces; r += kThreads)
    sh_h[r] = randomk_hash(S.hash, step, S.part, rankterms[S.piece0 + r]);
  __syncthreads();
  for (int j = 0; j < kUnit / (kThreads * 4); ++j) {
    const uint32_t e = u * kUnit + (j * kThreads + threadIdx.x) * 4;
    if (e >= n) break;
    const uint32_t last = min(e + 3, n - 1);
    const uint64_t j0 = stratum_of(e, k, n), j1 = stratum_of(last, k, n);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t r = 0; r < S.npieces; ++r) {
      const float* val = reinterpret_cast<const float*>(pieces[S.piece0 + r]);
      const uint64_t h = sh_h[r];
      for (uint64_t jj = j0; jj <= j1; ++jj) {
        const uint32_t idx = randomk_pick(h, jj, k, n);
        if (idx >= e && idx <= last) {
          const int c = idx - e;
          f4set(acc, c, __fadd_rn(f4get(acc, c), __ldg(val + jj)));
        }
      }
    }
    if (S.divisor != 1.0f && (acc.x != 0.f || acc.y != 0.f || acc.z != 0.f || acc.w != 0.f))
      acc = Divisor(S.divisor)(acc);
    store4_guard(seg_out(S), e, n, acc);
  }
}

// The h1 on the persistent TMA streaming driver: per run of 512 elements,
// acc = g + r, the hashed pick of each stratum touching a float4, r := sel ? 0 : acc.
struct RandomkOp {
  struct State {
    uint64_t h;
  };
  __device__ void begin_segment(const SegH1& S, State& st, TmaHdr&) const {
    st.h = randomk_hash(S.hash, *S.step, S.part, S.rankterm);
  }
  const unsigned char* const* pieces = nullptr;   // not a decoding op
  template <bool FULL>
  __device__ void run(const SegH1& S, const float4 (&gv)[kNJ], const float4 (&rv)[kNJ], uint32_t base,
                      State& st, TmaHdr&, const uint32_t*) const {
    const uint32_t n = S.n, k = S.k;
    if (base >= n) return;
    const int lane = threadIdx.x & 31;
    float* val = reinterpret_cast<float*>(S.chunk);
#pragma unroll
    for (int j = 0; j < kNJ; ++j) {
      const uint32_t e = base + j * 128 + lane * 4;
      if (e >= n) continue;
      float4 acc = gv[j];
      if (S.ef) {
        acc.x = __fadd_rn(acc.x, rv[j].x);
        acc.y = __fadd_rn(acc.y, rv[j].y);
        acc.z = __fadd_rn(acc.z, rv[j].z);
        acc.w = __fadd_rn(acc.w, rv[j].w);
      }
      const uint32_t last = min(e + 3, n - 1);
      const uint64_t j0 = stratum_of(e, k, n), j1 = stratum_of(last, k, n);
      uint32_t sel = 0;
      for (uint64_t jj = j0; jj <= j1; ++jj) {
        const uint32_t idx = randomk_pick(st.h, jj, k, n);
        if (idx >= e && idx <= last) {
          sel |= 1u << (idx - e);
          val[jj] = f4get(acc, idx - e);
        }
      }
      if (S.ef) {
        float4 nr = acc;
        if (sel & 1) nr.x = 0.f;
        if (sel & 2) nr.y = 0.f;
        if (sel & 4) nr.z = 0.f;
        if (sel & 8) nr.w = 0.f;
        store4_guard(S.r, e, n, nr);
      }
    }
  }
  __device__ void end_segment(const SegH1&, uint32_t, uint32_t, State&, TmaHdr&) const {}
};

int tma_stream_grid(int nunits);
int tma_stream_stages();

void launch_randomk_h1(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st) {
  if (nunits == 0) return;
  static bool init = [] {
    return cudaFuncSetAttribute(tma_stream_kernel<RandomkOp>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kTmaHdrBytes + kTmaMaxStages * kTmaStageBytes)) == cudaSuccess;
  }();
  (void)init;
  const int ns = tma_stream_stages();
  tma_stream_kernel<<<tma_stream_grid(nunits), kThreads + 32, kTmaHdrBytes + ns * kTmaStageBytes, st>>>(
      segs, unit_seg, (uint32_t)nunits, ns, RandomkOp{});
  count_launches(1);
}

void launch_h2_randomk(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                       const unsigned char* const* pieces, const uint32_t* rankterms, cudaStream_t st) {
  if (nunits == 0) return;
  h2_randomk_kernel<<<nunits, kThreads, 0, st>>>(segs, unit_seg, pieces, rankterms);
  count_launches(1);
}

}  // namespace esp
