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
// h2: per 1024-element tile (one warp), zero fill, then each stratum's
// pick(s) written once with the rank-order sum of the pieces' values (÷ n).
#include "esp_device.cuh"
#include "esp_kernels.h"
#include "stream_tma.cuh"

namespace esp {

// floor(x / d) for d >= 1 and a quotient below 2^32 (x < 2^64): a double
// estimate -- relative error below 3 * 2^-53, so within 1 of the quotient --
// corrected in integers.  Exact, like the 64-bit division it replaces (a
// ~70-instruction software routine; the picks are a few % of the h2 pass).
__device__ __forceinline__ uint64_t div_q32(uint64_t x, uint64_t d, double inv_d) {
  uint64_t q = __double2ull_rz(__dmul_rn(__ull2double_rn(x), inv_d));
  const int64_t r = (int64_t)(x - q * d);   // in (-d, 2d)
  if (r < 0) --q;
  else if ((uint64_t)r >= d) ++q;
  return q;
}

// The divisions of a segment's strata, n and k fixed: stratum j is
// [floor(j n / k), floor((j + 1) n / k)), of length floor(n / k) or one more.
struct StrataDiv {
  uint32_t n, k;
  double inv_n, inv_k;
  __device__ __forceinline__ void init(uint32_t n_, uint32_t k_) {
    n = n_;
    k = k_ ? k_ : 1u;
    inv_n = __drcp_rn((double)n);
    inv_k = __drcp_rn((double)k);
  }
  // the stratum holding element i: ceil((i + 1) k / n) - 1
  __device__ __forceinline__ uint64_t stratum_of(uint64_t i) const {
    return div_q32((i + 1) * k + n - 1, n, inv_n) - 1;
  }
  __device__ __forceinline__ uint64_t start(uint64_t j) const { return div_q32(j * n, k, inv_k); }
  // h mod len: (hi mod len) 2^32 + lo < len 2^32, each step a quotient < 2^32
  __device__ __forceinline__ static uint64_t mod(uint64_t h, uint64_t len) {
    const double inv = __drcp_rn((double)len);
    const uint64_t hi = h >> 32;
    const uint64_t x = ((hi - div_q32(hi, len, inv) * len) << 32) | (h & 0xFFFFFFFFull);
    return x - div_q32(x, len, inv) * len;
  }
  // the pick of stratum j under hash h (reading R5): start_j + mix(h ^ j) mod len_j
  __device__ __forceinline__ uint32_t pick(uint64_t h, uint64_t j) const {
    const uint64_t a = start(j), b = start(j + 1);
    return (uint32_t)(a + mod(splitmix64(h ^ j), b - a));
  }
};

// The oracle's chain (reading R5): h = mix(mix(mix(mix(mix(seed)^tensor)^step)^part)^rankterm),
// pick_j = start_j + mix(h ^ j) mod len_j.  `base` = mix(mix(seed)^tensor) from the planner.
__device__ __forceinline__ uint64_t randomk_hash(uint64_t base, uint64_t step, uint32_t part,
                                                  uint32_t rankterm) {
  return splitmix64(splitmix64(splitmix64(base ^ step) ^ (uint64_t)part) ^ (uint64_t)rankterm);
}


// ------------------------------------------------------------------ h1
struct RandomkOp {
  static constexpr int kGroups = 3;   // consumer groups
  struct State {
    uint64_t h;
    StrataDiv sd;
  };
  const unsigned char* const* pieces = nullptr;   // not a decoding op
  bool stage_words = false;
  template <int BAR>
  __device__ void begin_segment(const SegH1& S, State& st, TmaGroup&) const {
    st.h = randomk_hash(S.hash, *S.step, S.part, S.rankterm);
    st.sd.init(S.n, S.k);
  }
  template <bool FULL>
  __device__ void run(const SegH1& S, const float4 (&gv)[kNJ], const float4 (&rv)[kNJ], uint32_t base,
                      State& st, TmaGroup& hd, const uint32_t*) const {
    const uint32_t n = S.n;
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
    const uint64_t j0 = st.sd.stratum_of(base), j1 = st.sd.stratum_of(hi);
    float* val = reinterpret_cast<float*>(S.chunk);
    for (uint64_t jb = j0; jb <= j1; jb += 32) {
      const uint64_t jj = jb + lane;
      if (jj <= j1) {
        const uint32_t p = st.sd.pick(st.h, jj);
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
// its own hash (identical for all pieces when indices are shared).  One WARP
// per 1024-element output tile (8 per 8192-element unit of the unit table),
// persistent over tiles, no CTA barrier: the tile is zero-filled from
// registers (the 4 B/elem write that bounds the kernel), then every stratum
// overlapping the tile gets one lane, which computes its pick(s) and writes
// the rank-order sum from +0 of the pieces' values at each picked position
// inside the tile (a boundary stratum is evaluated by both neighbouring tiles;
// each writes only its own positions, so zero fill and picks of a position
// are ordered within one warp).  Strata are disjoint ranges, so a position
// can only be picked by ONE stratum, whatever the piece.
constexpr int kRkBatch = 8;
constexpr int kRkTile = 1024;
__global__ void __launch_bounds__(kTileThreads) h2_randomk_kernel(const SegH2* __restrict__ segs,
                                                                  const uint32_t* __restrict__ unit_seg,
                                                                  uint32_t nunits,
                                                                  const unsigned char* const* __restrict__ pieces,
                                                                  const uint32_t* __restrict__ rankterms) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  constexpr int kWarps = kTileThreads / 32;
  constexpr int kSub = kUnit / kRkTile;
  constexpr unsigned kFull = 0xffffffffu;
  __shared__ uint64_t sh_h[kWarps][64];
  __shared__ const float* sh_v[kWarps][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* hh = sh_h[warp];
  const float** vv = sh_v[warp];
  const uint32_t ntiles = nunits * kSub, GW = gridDim.x * kWarps;
  uint32_t cur = 0xFFFFFFFFu;
  SegH2 S{};
  StrataDiv sd{};
  bool shared = true;
  for (uint32_t gt = blockIdx.x * kWarps + warp; gt < ntiles; gt += GW) {
    const uint32_t unit = gt / kSub;
    const uint32_t sid = unit_seg[unit];
    if (sid != cur) {
      cur = sid;
      S = segs[sid];
      sd.init(S.n, S.k);
      const uint64_t step = *S.step;
      __syncwarp();   // the previous segment's tables are no longer read
      for (uint32_t r = lane; r < S.npieces; r += 32) {
        hh[r] = randomk_hash(S.hash, step, S.part, rankterms[S.piece0 + r]);
        vv[r] = reinterpret_cast<const float*>(pieces[S.piece0 + r]);
      }
      __syncwarp();
      bool same = true;
      for (uint32_t r = lane; r < S.npieces; r += 32) same &= hh[r] == hh[0];
      shared = __all_sync(kFull, same);
    }
    const uint32_t n = S.n, np = S.npieces;
    const uint32_t lo = (unit - S.unit0) * kUnit + (gt % kSub) * kRkTile;
    if (lo >= n) continue;   // past the segment's last element (warp-uniform)
    const uint32_t hi = min(lo + (uint32_t)kRkTile, n) - 1;
    float* out = seg_out(S);
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hi + 1 - lo == (uint32_t)kRkTile && al16(out + lo)) {
#pragma unroll
      for (int j = 0; j < kRkTile / 128; ++j) st4(out + lo + lane * 4 + 128 * j, z);
    } else {
      for (uint32_t i = lo + lane * 4; i <= hi; i += 128) store4_guard(out, i, n, z);
    }
    __syncwarp();   // zero stores before the picks' stores
    const Divisor div(S.divisor);
    const bool ones = S.divisor == 1.0f;
    const uint64_t j0 = sd.stratum_of(lo), j1 = sd.stratum_of(hi);
    for (uint64_t jj = j0 + lane; jj <= j1; jj += 32) {
      const uint64_t a = sd.start(jj), len = sd.start(jj + 1) - a;
      auto pick = [&](uint32_t r) { return (uint32_t)(a + sd.mod(splitmix64(hh[r] ^ jj), len)); };
      if (shared) {
        const uint32_t p = pick(0);
        if (p < lo || p > hi) continue;
        float sum = 0.f;
        for (uint32_t r0 = 0; r0 < np; r0 += kRkBatch) {
          float v[kRkBatch];
#pragma unroll
          for (int m = 0; m < kRkBatch; ++m) v[m] = r0 + m < np ? __ldg(vv[r0 + m] + jj) : 0.f;
#pragma unroll
          for (int m = 0; m < kRkBatch; ++m)
            if (r0 + m < np) sum = __fadd_rn(sum, v[m]);
        }
        out[p] = ones ? sum : div(sum);
      } else {
        // per-rank indices: the pieces' picks of this stratum; each distinct
        // position inside the tile gets the rank-order sum of its pieces
        for (uint32_t r = 0; r < np; ++r) {
          const uint32_t p = pick(r);
          if (p < lo || p > hi) continue;
          bool first = true;
          for (uint32_t q = 0; q < r && first; ++q) first = pick(q) != p;
          if (!first) continue;   // written with an earlier piece's pick
          float sum = __fadd_rn(0.f, __ldg(vv[r] + jj));
          for (uint32_t q = r + 1; q < np; ++q)
            if (pick(q) == p) sum = __fadd_rn(sum, __ldg(vv[q] + jj));
          out[p] = ones ? sum : div(sum);
        }
      }
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2_randomk_kernel, kTileThreads, 0);
    return sms * (per_sm > 0 ? per_sm : 8);
  }();
  const int need = (nunits * (kUnit / kRkTile) + kTileThreads / 32 - 1) / (kTileThreads / 32);   // a warp per tile
  const int grid = need < cap ? need : cap;
  launch_pdl(h2_randomk_kernel, grid, kTileThreads, 0, st, segs, unit_seg, (uint32_t)nunits, pieces, rankterms);
  count_launches(1);
}

}  // namespace esp
