// h2 on sm_100a: fused decompression + aggregation of the n (Allgather) or
// n^2 (Alltoall/Allgather) received pieces, written once into the gradient
// ("fuses the decompression operations"; n h2(M) and n^2 h2(M/n) of the
// cost table).
//
// Aggregation rule (reading R9): fp32 sum over pieces in rank order starting
// from +0.0f, then IEEE division by the divisor (n for MEAN).  Adding an
// implicit +0 for an absent sparse entry is the identity on a sum that started
// at +0.0f, so the sparse kernel only touches present entries.
#include <algorithm>

#include "esp_device.cuh"
#include "esp_kernels.h"

namespace esp {

constexpr int kMaxPieces = 64;

// For every piece (sorted idx[kpad], 0xFFFFFFFF padding), the first entry of
// each output tile: toff[t] = lower_bound(idx, t * kTile), t = 0..ntiles.  One
// pass over the (small) pieces replaces a dependent binary search per tile.
// job = {segment, piece within segment, first entry}: kOffJob entries of one
// piece; every thread issues all of its loads (its entries and their
// predecessors) before using any (the loop was a chain of dependent loads).
__global__ void __launch_bounds__(kThreads) h2_sparse_offsets_kernel(const SegH2* __restrict__ segs,
                                                                     const uint4* __restrict__ jobs,
                                                                     const unsigned char* const* __restrict__ pieces) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  constexpr int kPer = kOffJob / kThreads;
  const uint4 job = jobs[blockIdx.x];
  const SegH2 S = segs[job.x];
  const uint32_t r = job.y;
  const uint32_t ntiles = S.nunits;
  uint32_t* toff = S.toff + (size_t)r * (ntiles + 1);
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(pieces[S.piece0 + r]);
  const uint32_t iend = min(job.z + (uint32_t)kOffJob, S.kpad);
  auto tile_of = [&](uint32_t v) { return v == 0xFFFFFFFFu ? ntiles : min(v / (uint32_t)kTile, ntiles); };
  uint32_t v[kPer], u[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const uint32_t i = job.z + threadIdx.x + q * kThreads;
    v[q] = i < iend ? __ldg(idx + i) : 0u;
    u[q] = (i < iend && i > 0) ? __ldg(idx + i - 1) : 0u;
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const uint32_t i = job.z + threadIdx.x + q * kThreads;
    if (i >= iend) break;
    const uint32_t t = tile_of(v[q]);
    const uint32_t prev = i == 0 ? 0u : tile_of(u[q]) + 1;
    for (uint32_t qq = prev; qq <= t; ++qq) toff[qq] = i;   // tiles (tile(i-1), tile(i)] start at i
    if (i == S.kpad - 1)
      for (uint32_t qq = t + 1; qq <= ntiles; ++qq) toff[qq] = S.kpad;
  }
}

// A warp's zero fill of out[lo, hi) (one 1024-element tile): eight unrolled
// 16-byte stores per lane for a full aligned tile, else guarded.
__device__ __forceinline__ void zero_tile(float* out, uint32_t lo, uint32_t hi, uint32_t n) {
  const int lane = threadIdx.x & 31;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (hi - lo == (uint32_t)kTile && al16(out + lo)) {
#pragma unroll
    for (int j = 0; j < kTile / 128; ++j) st4(out + lo + lane * 4 + 128 * j, z);
  } else {
    for (uint32_t i = lane * 4; lo + i < hi; i += 128) store4_guard(out, lo + i, n, z);
  }
}

// One WARP per output tile, persistent over tiles (stride = all warps of the
// grid): no CTA barrier anywhere, so 64 independent tiles per SM hide the load
// latencies of the entry lists (a CTA-wide tile loop was latency-bound).
// Per tile, by the number of entries the pieces have in it:
//   one piece:     dense zero fill straight from registers (the 4 B/elem write
//                  that bounds the kernel), then out[e] = (+0 + v) / d for the
//                  touched words;
//   several, <= 32 entries in the tile (the sparse common case): zero fill, then
//                  one entry per lane, equal indices grouped by
//                  __match_any_sync, each group summed from +0 in lane (= rank)
//                  order by its lowest lane and stored once;
//   several, more: the warp's 1024-float shared-memory tile starts at +0; the
//                  entries in rank-major order are added 32 per round (equal
//                  indices within a round grouped as above, summed in lane =
//                  rank order onto the earlier rounds' value); then the tile is
//                  divided and written once with coalesced float4 stores -- no
//                  global read-modify-write.
// MULTI = false (every segment of the launch has one piece, e.g. a single
// rank's payload): only the zero fill + touched-word path, no shared memory
// (assembling dense tiles in shared memory measured slower on BERT-large).
template <bool MULTI>
__global__ void __launch_bounds__(kTileThreads, MULTI ? 8 : 1) h2_sparse_kernel(const SegH2* __restrict__ segs,
                                                                 const uint32_t* __restrict__ tile_seg,
                                                                 uint32_t ntiles,
                                                                 const unsigned char* const* __restrict__ pieces) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  constexpr int kWarps = kTileThreads / 32;
  constexpr unsigned kFull = 0xffffffffu;
  // the per-warp 4 KB accumulation tiles (dynamic shared memory, MULTI only)
  extern __shared__ __align__(16) float acc_all[];
  const int lane = threadIdx.x & 31;
  float* acc = acc_all + (threadIdx.x >> 5) * kTile;
  const uint32_t GW = gridDim.x * kWarps;
  uint32_t tg = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (tg >= ntiles) return;
  SegH2 S = segs[tile_seg[tg]];
  float* out = seg_out(S);
  // lane holds the entry range of pieces lane and lane + 32 for the current tile
  uint32_t plo0 = 0, phi0 = 0, plo1 = 0, phi1 = 0;
  auto load_toff = [&](const SegH2& s, uint32_t t) {
    if ((uint32_t)lane < s.npieces) {
      const uint32_t* toff = s.toff + (size_t)lane * (s.nunits + 1) + t;
      plo0 = __ldg(toff);
      phi0 = __ldg(toff + 1);
    }
    if ((uint32_t)lane + 32 < s.npieces) {
      const uint32_t* toff = s.toff + (size_t)(lane + 32) * (s.nunits + 1) + t;
      plo1 = __ldg(toff);
      phi1 = __ldg(toff + 1);
    }
  };
  load_toff(S, tg - S.unit0);
  // lane r holds the pointers of pieces r and r + 32 of the current segment
  const unsigned char* pp0 = nullptr;
  const unsigned char* pp1 = nullptr;
  auto load_pp = [&](const SegH2& s) {
    if ((uint32_t)lane < s.npieces) pp0 = pieces[s.piece0 + lane];
    if ((uint32_t)lane + 32 < s.npieces) pp1 = pieces[s.piece0 + lane + 32];
  };
  load_pp(S);
  while (true) {
    const uint32_t t = tg - S.unit0;
    const uint32_t lo = t * kTile;
    const uint32_t hi = min(lo + (uint32_t)kTile, S.n);
    const uint32_t np = S.npieces;
    const bool ones = S.divisor == 1.0f;
    const Divisor div(S.divisor);
    const uint32_t clo0 = plo0, chi0 = phi0, clo1 = plo1, chi1 = phi1;
    auto range = [&](uint32_t r, uint32_t* a, uint32_t* b) {
      *a = __shfl_sync(kFull, r < 32 ? clo0 : clo1, r & 31);
      *b = __shfl_sync(kFull, r < 32 ? chi0 : chi1, r & 31);
    };
    // the next tile (same segment unless past its last tile): offsets in flight
    // while this tile's entries are processed
    const uint32_t tn = tg + GW;
    const SegH2* Sn_p = nullptr;
    if (tn < ntiles) {
      if (tn >= S.unit0 + S.nunits) Sn_p = segs + tile_seg[tn];
      load_toff(Sn_p ? *Sn_p : S, tn - (Sn_p ? Sn_p->unit0 : S.unit0));
    }
    // the tile's entries of all pieces, in rank order: lane l takes the l-th
    uint32_t tot = 0, my_r = 0xFFFFFFFFu, my_i = 0;
    if (MULTI && np > 1) {
      for (uint32_t r = 0; r < np; ++r) {
        uint32_t a, b;
        range(r, &a, &b);
        if ((uint32_t)lane >= tot && (uint32_t)lane < tot + (b - a)) {
          my_r = r;
          my_i = a + (lane - tot);
        }
        tot += b - a;
      }
    }
    if (MULTI && np > 1 && tot > 32) {
      // shared-memory accumulation in rank order, one coalesced write.  The
      // tile's entries in rank-major order (piece, then index) are taken 32 per
      // round, kRounds rounds' loads in flight at once; inside a round the
      // lanes holding one index form a group (__match_any_sync) whose lowest
      // lane adds the members' values in lane (= rank) order to the tile value
      // left by the earlier rounds (= lower ranks); __syncwarp between rounds.
#pragma unroll
      for (int i = lane * 4; i < kTile; i += 128)
        *reinterpret_cast<float4*>(acc + i) = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
      constexpr int kRounds = 3;
      for (uint32_t x0 = 0; x0 < tot; x0 += 32 * kRounds) {
        uint32_t pr[kRounds], li[kRounds];   // piece and entry of position x0 + 32 q + lane
#pragma unroll
        for (int q = 0; q < kRounds; ++q) pr[q] = 0xFFFFFFFFu;
        uint32_t start = 0;
        for (uint32_t r = 0; r < np; ++r) {
          uint32_t a, b;
          range(r, &a, &b);
#pragma unroll
          for (int q = 0; q < kRounds; ++q) {
            const uint32_t x = x0 + 32 * q + lane;
            if (x - start < b - a) { pr[q] = r; li[q] = a + (x - start); }   // unsigned: start <= x < start + cnt
          }
          start += b - a;
        }
        uint32_t e[kRounds];
        float v[kRounds];
#pragma unroll
        for (int q = 0; q < kRounds; ++q) {
          const uint32_t r = pr[q] == 0xFFFFFFFFu ? 0u : pr[q];
          const unsigned char* pc = reinterpret_cast<const unsigned char*>(
              __shfl_sync(kFull, reinterpret_cast<unsigned long long>(r < 32 ? pp0 : pp1), r & 31));
          e[q] = 0x80000000u | (uint32_t)lane;   // no entry: a key no index has
          v[q] = 0.f;
          if (pr[q] != 0xFFFFFFFFu) {
            e[q] = __ldg(reinterpret_cast<const uint32_t*>(pc) + li[q]);
            v[q] = __ldg(reinterpret_cast<const float*>(pc + 4 * (size_t)S.kpad) + li[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < kRounds; ++q) {
          if (x0 + 32 * q >= tot) break;   // warp-uniform
          const bool mine = pr[q] != 0xFFFFFFFFu;
          const uint32_t grp = __match_any_sync(kFull, e[q]);
          const bool lead = mine && __ffs(grp) - 1 == lane;
          const int gmax = __reduce_max_sync(kFull, (uint32_t)__popc(grp));
          float s = lead ? acc[e[q] - lo] : 0.f;
          uint32_t rest = grp;
          for (int m = 0; m < gmax; ++m) {
            const float y = __shfl_sync(kFull, v[q], rest ? __ffs(rest) - 1 : lane);
            if (rest) {
              s = __fadd_rn(s, y);
              rest &= rest - 1;
            }
          }
          if (lead) acc[e[q] - lo] = s;
          __syncwarp();
        }
      }
      for (uint32_t i = lane * 4; lo + i < hi; i += 128) {
        float4 v = *reinterpret_cast<const float4*>(acc + i);
        if (!ones) v = div(v);
        store4_guard(out, lo + i, S.n, v);
      }
    } else if (!MULTI || np == 1) {
      // one piece: zero fill from registers, then the touched words
      const unsigned char* pc = pieces[S.piece0];
      const uint32_t* idx = reinterpret_cast<const uint32_t*>(pc);
      const float* val = reinterpret_cast<const float*>(pc + 4 * (size_t)S.kpad);
      uint32_t a, b;
      range(0, &a, &b);
      zero_tile(out, lo, hi, S.n);
      __syncwarp();   // zero stores before the touched-word stores
      for (uint32_t i = a + lane; i < b; i += 32) {
        const float v = __fadd_rn(0.f, __ldg(val + i));   // +0 + v: the oracle's sum from +0
        out[__ldg(idx + i)] = ones ? v : div(v);
      }
    } else {
      zero_tile(out, lo, hi, S.n);
      __syncwarp();   // zero stores before the touched-word stores
      {
        // one entry per lane: lanes holding the same index form a group
        // (__match_any_sync), whose lowest lane sums it in lane = rank order
        // from +0 and stores it once -- no read-modify-write round trips
        const int src = (int)(my_r & 31u);
        const unsigned char* q0 = reinterpret_cast<const unsigned char*>(
            __shfl_sync(kFull, reinterpret_cast<unsigned long long>(pp0), src));
        const unsigned char* q1 = reinterpret_cast<const unsigned char*>(
            __shfl_sync(kFull, reinterpret_cast<unsigned long long>(pp1), src));
        uint32_t e = 0x80000000u | (uint32_t)lane;   // no entry: a key no index has
        float v = 0.f;
        if (my_r != 0xFFFFFFFFu) {
          const unsigned char* pc = my_r < 32 ? q0 : q1;
          e = __ldg(reinterpret_cast<const uint32_t*>(pc) + my_i);
          v = __ldg(reinterpret_cast<const float*>(pc + 4 * (size_t)S.kpad) + my_i);
        }
        const uint32_t grp = __match_any_sync(kFull, e);
        float sum = 0.f;
        uint32_t rest = grp;
        for (uint32_t m = 0; m < np; ++m) {   // at most one member per piece
          const float x = __shfl_sync(kFull, v, rest ? __ffs(rest) - 1 : lane);
          if (rest) {
            sum = __fadd_rn(sum, x);
            rest &= rest - 1;
          }
        }
        if (my_r != 0xFFFFFFFFu && __ffs(grp) - 1 == lane) out[e] = ones ? sum : div(sum);
      }
    }
    if (tn >= ntiles) break;
    tg = tn;
    if (Sn_p) {
      S = *Sn_p;
      out = seg_out(S);
      load_pp(S);
    }
    __syncwarp();   // shared tile reuse
  }
}

// first position in idx[0, len) holding a value >= target (sorted, warp-wide)
__device__ __forceinline__ uint32_t warp_lower_bound(const uint32_t* idx, uint32_t len, uint32_t target) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = len;   // idx[< lo] < target <= idx[>= hi]
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t p = lo + lane * step;
    const bool below = p < hi && __ldg(idx + p) < target;
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, below));   // probes below: lanes 0..c-1
    const uint32_t nlo = c ? lo + (c - 1) * step + 1 : lo;
    const uint32_t nhi = lo + c * step < hi ? lo + c * step : hi;
    lo = nlo;
    hi = nhi;
  }
  const bool below = lo + lane < hi && __ldg(idx + lo + lane) < target;
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// One piece per segment (a single rank's payload, an NCCL-reduced bucket's
// unpack): one WARP per contiguous range of 1024-element tiles, persistent,
// no tile-offset pass.  The warp keeps a cursor into the piece's sorted
// entries (a 32-ary lower_bound only where its range starts inside a
// segment); per tile it issues the next 32 entries' loads, zero-fills the tile
// from registers (eight 16-byte stores per lane), then stores the tile's
// entries (those below the tile's end; more batches for dense tiles) as
// out[e] = (+0 + v) / d and advances the cursor.
__global__ void __launch_bounds__(kTileThreads) h2_sparse1_kernel(const SegH2* __restrict__ segs,
                                                                 const uint32_t* __restrict__ tile_seg,
                                                                 uint32_t ntiles,
                                                                 const unsigned char* const* __restrict__ pieces) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  constexpr int kWarps = kTileThreads / 32;
  const int lane = threadIdx.x & 31;
  const uint32_t W = gridDim.x * kWarps, wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t t0 = (uint32_t)((uint64_t)wid * ntiles / W), t1 = (uint32_t)((uint64_t)(wid + 1) * ntiles / W);
  uint32_t cur_seg = 0xFFFFFFFFu, cur = 0;
  SegH2 S{};
  const uint32_t* idx = nullptr;
  const float* val = nullptr;
  // a batch of 32 entries in registers, lane l holding entry bb + l: refilled
  // only when consumed (a sparse tile uses one or two of them), so most tiles
  // issue no dependent load at all
  uint32_t bb = 0, e = 0xFFFFFFFFu;
  float v = 0.f;
  auto refill = [&](uint32_t at) {
    bb = at;
    const uint32_t q = at + lane;
    e = q < S.kpad ? __ldg(idx + q) : 0xFFFFFFFFu;   // padding entries are 0xFFFFFFFF
    v = q < S.kpad ? __ldg(val + q) : 0.f;
  };
  uint32_t sid_next = t0 < t1 ? tile_seg[t0] : 0u;
  for (uint32_t t = t0; t < t1; ++t) {
    const uint32_t sid = sid_next;
    if (t + 1 < t1) sid_next = tile_seg[t + 1];
    if (sid != cur_seg) {
      cur_seg = sid;
      S = segs[sid];
      const unsigned char* pc = pieces[S.piece0];
      idx = reinterpret_cast<const uint32_t*>(pc);
      val = reinterpret_cast<const float*>(pc + 4 * (size_t)S.kpad);
      cur = t == S.unit0 ? 0u : warp_lower_bound(idx, S.kpad, (t - S.unit0) * kTile);
      refill(cur);
    }
    const uint32_t lo = (t - S.unit0) * kTile, hi = min(lo + (uint32_t)kTile, S.n);
    float* out = seg_out(S);
    zero_tile(out, lo, hi, S.n);
    __syncwarp();   // zero stores before the touched-word stores
    const bool ones = S.divisor == 1.0f;
    const Divisor div(S.divisor);
    while (true) {
      const bool in = bb + lane >= cur && e < hi;   // sorted: the tile's entries come first
      if (in) {
        const float x = __fadd_rn(0.f, v);   // +0 + v: the oracle's sum from +0
        out[e] = ones ? x : div(x);
      }
      cur += __popc(__ballot_sync(0xffffffffu, in));
      if (cur < bb + 32) break;   // entries left in the batch belong to later tiles
      refill(cur);                // consumed: the next 32 (more of this tile, or later ones)
    }
  }
}

// Several pieces, dense tiles (expected > 32 entries per 1024 elements, e.g.
// DGC 1% at n >= 4): one CTA per 8192-element tile, persistent over a
// CONTIGUOUS range of tiles, assembled in a 32 KB shared-memory accumulator:
// zero fill; warp w streams piece pc + w's entries from a cursor (the
// entries are sorted by index: those below the tile's end are the tile's, the
// rest stay for the next tile -- no tile-offset pass; one warp-wide 32-ary
// lower_bound per piece where a CTA starts inside a segment); the pieces are
// added in rank order, one CTA phase per piece (indices are distinct within a
// piece, so a phase has no conflicts); then divided and written once with
// coalesced stores.
constexpr int kCtaTile = 8 * kTile;
__global__ void __launch_bounds__(kThreads, 5) h2_sparse_cta_kernel(const SegH2* __restrict__ segs,
                                                                    const uint32_t* __restrict__ tile_seg,
                                                                    uint32_t ntiles,
                                                                    const unsigned char* const* __restrict__ pieces) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  __shared__ __align__(16) float acc[kCtaTile];
  __shared__ uint32_t sh_cur[kMaxPieces];   // per piece: the next entry not yet consumed
  constexpr int L = 4;   // entries per lane in flight
  constexpr int kW = kThreads / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t nct = (ntiles + 7) / 8;
  const uint32_t c0 = (uint32_t)((uint64_t)blockIdx.x * nct / gridDim.x);
  const uint32_t c1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * nct / gridDim.x);
  uint32_t cur_seg = 0xFFFFFFFFu;
  for (uint32_t t = c0 * 8; t < min(c1 * 8, ntiles);) {
    const uint32_t tend = min(c1 * 8, ntiles);
    const uint32_t sid = tile_seg[t];
    const SegH2 S = segs[sid];
    const uint32_t u0 = t - S.unit0;
    const uint32_t u1 = min(min(tend, S.unit0 + S.nunits), (t & ~7u) + 8) - S.unit0;   // one CTA tile at most
    t = S.unit0 + u1;
    const uint32_t lo = u0 * kTile, hi = min(u1 * kTile, S.n), len = hi - lo;   // elements [lo, hi)
    const uint32_t np = S.npieces;
    if (sid != cur_seg) {   // a new segment: the cursors at lo (0 at the segment's start)
      cur_seg = sid;
      __syncthreads();   // the previous segment's cursors are no longer read
      for (uint32_t r = w; r < np; r += kW) {
        const uint32_t c = u0 == 0 ? 0u : warp_lower_bound(reinterpret_cast<const uint32_t*>(pieces[S.piece0 + r]), S.kpad, lo);
        if (lane == 0) sh_cur[r] = c;
      }
    }
    for (uint32_t i = threadIdx.x * 4; i < len; i += kThreads * 4)
      *reinterpret_cast<float4*>(acc + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();   // zero fill and cursors
    for (uint32_t pc = 0; pc < np; pc += kW) {
      const uint32_t r = pc + w;
      const uint32_t* idx = nullptr;
      const float* val = nullptr;
      uint32_t a = 0;
      if (r < np) {
        const unsigned char* pr = pieces[S.piece0 + r];
        idx = reinterpret_cast<const uint32_t*>(pr);
        val = reinterpret_cast<const float*>(pr + 4 * (size_t)S.kpad);
        a = sh_cur[r];
      }
      uint32_t e[L];
      float v[L];
#pragma unroll
      for (int m = 0; m < L; ++m) {
        const uint32_t q = a + lane + 32 * m;
        e[m] = (r < np && q < S.kpad) ? __ldg(idx + q) : 0xFFFFFFFFu;   // (padding entries are 0xFFFFFFFF)
        v[m] = (r < np && q < S.kpad) ? __ldg(val + q) : 0.f;
      }
      for (uint32_t p = 0; p < (uint32_t)kW && pc + p < np; ++p) {
        if ((uint32_t)w == p) {
          uint32_t used = 0;
          bool more = true;
#pragma unroll
          for (int m = 0; m < L; ++m) {
            const bool in = e[m] < hi;   // sorted: the tile's entries come first
            if (in) acc[e[m] - lo] = __fadd_rn(acc[e[m] - lo], v[m]);
            const uint32_t bm = __ballot_sync(0xffffffffu, in);
            used += __popc(bm);
            more = more && bm == 0xffffffffu;
          }
          for (uint32_t q0 = a + 32 * L; more; q0 += 32) {   // dense tiles (TOPK, large ratios)
            const uint32_t q = q0 + lane;
            const uint32_t x = q < S.kpad ? __ldg(idx + q) : 0xFFFFFFFFu;
            const bool in = x < hi;
            if (in) acc[x - lo] = __fadd_rn(acc[x - lo], __ldg(val + q));
            const uint32_t bm = __ballot_sync(0xffffffffu, in);
            used += __popc(bm);
            more = bm == 0xffffffffu;
          }
          if (lane == 0) sh_cur[r] = a + used;
        }
        __syncthreads();
      }
    }
    const bool ones = S.divisor == 1.0f;
    const Divisor div(S.divisor);
    float* out = seg_out(S);
    for (uint32_t i = threadIdx.x * 4; i < len; i += kThreads * 4) {
      float4 x = *reinterpret_cast<const float4*>(acc + i);
      if (!ones) x = div(x);
      store4_guard(out, lo + i, S.n, x);
    }
    __syncthreads();   // the accumulator is read before the next tile's zero fill
  }
}

// Sign h2: a grid of a few CTAs per SM, each over a contiguous range of the
// bucket's units (mostly inside one segment), so the dependent prologue of a
// segment (its table entry, the piece pointers and scales) is paid once per
// (CTA, segment) instead of once per unit.  A unit is 8192 elements (256
// words = 1 KB per piece); a thread decodes 8 float4 of it.  Rank-order fp32
// sum from +0 over the pieces, then / divisor (R9), by one of:
//  * 1 piece: the words straight from global memory into registers, the next
//    unit's already in flight while this one is decoded (a select per element);
//  * 2..8 pieces: the words of all pieces staged in shared memory with
//    coalesced 16-byte loads (one round trip per unit, the next unit's in
//    flight), and the decoded sum looked up by bit pattern (esp_device.cuh)
//    in a table replicated 32 times, [pattern][lane], so that the 32 lanes'
//    random lookups never share a bank;
//  * more pieces: staged words, sequential select + add per piece.
constexpr int kSignWords = kSignUnit / 32;           // words per piece and unit
constexpr int kSignVec = kSignWords / 4;             // uint4 per piece and unit
constexpr int kSignPre = 4;                          // uint4 per thread in flight (pieces <= 16)
constexpr int kSignLutBytes = (1 << kSignLutPieces) * 32 * 4;   // 32 KB
// staged word rows: 8 (zero rows for absent pieces) when the table path can run
__host__ __device__ constexpr int sign_h2_rows(int max_pieces) {
  return max_pieces < 2 ? 1 : (max_pieces < kSignLutPieces ? kSignLutPieces : max_pieces);
}
__host__ __device__ constexpr size_t sign_h2_smem(int max_pieces) {
  return (size_t)sign_h2_rows(max_pieces) * kSignWords * 4 + (max_pieces >= 2 ? kSignLutBytes : 0);
}
// 4 CTAs (32 warps) per SM: the output stream needs the stores of many warps
// in flight (126 registers and 2 CTAs per SM measured 4.5 TB/s)
template <int KIND>
__global__ void __launch_bounds__(kThreads, 4) h2_sign_kernel(const SegH2* __restrict__ segs,
                                                           const uint32_t* __restrict__ unit_seg,
                                                           uint32_t nunits,
                                                           const unsigned char* const* __restrict__ pieces,
                                                           int max_pieces) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  extern __shared__ __align__(16) uint32_t sh_dyn[];
  uint32_t* sh_words = sh_dyn;                                   // [npieces][kSignWords]
  float* sh_lut = reinterpret_cast<float*>(sh_dyn + sign_h2_rows(max_pieces) * kSignWords);   // [256][32]
  __shared__ float sh_sp[kMaxPieces], sh_sn[kMaxPieces];
  __shared__ const uint32_t* sh_w[kMaxPieces];
  constexpr int kJ = kSignUnit / (kThreads * 4);
  const int lane = threadIdx.x & 31;
  const uint32_t u0 = (uint32_t)((uint64_t)blockIdx.x * nunits / gridDim.x);
  const uint32_t u1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * nunits / gridDim.x);
  uint32_t cur = 0xFFFFFFFFu;
  SegH2 S{};
  // the next unit's words in flight, one register buffer for both paths:
  // staged paths: pre[m] = vector threadIdx.x + m * kThreads of the unit;
  // one piece: word j of this thread = component j % 4 of pre[j / 4]
  static_assert(kJ <= 4 * kSignPre, "one-piece words fit the prefetch buffer");
  uint4 pre[kSignPre];
  bool have = false;         // pre[] holds the words of unit gu
  uint32_t sid_next = u0 < u1 ? unit_seg[u0] : 0u;
  auto load_vec = [&](uint32_t v, uint32_t w0, uint32_t nwords) -> uint4 {
    const uint32_t r = v / kSignVec, q = v % kSignVec;
    const uint32_t w = w0 + q * 4;
    return w < nwords ? __ldg(reinterpret_cast<const uint4*>(sh_w[r] + w)) : make_uint4(0u, 0u, 0u, 0u);
  };
  for (uint32_t gu = u0; gu < u1; ++gu) {
    const uint32_t sid = sid_next;
    if (gu + 1 < u1) sid_next = unit_seg[gu + 1];
    if (sid != cur) {
      __syncthreads();   // the previous segment's tables and words are no longer read
      cur = sid;
      S = segs[sid];
      for (uint32_t r = threadIdx.x; r < S.npieces; r += kThreads) {
        const unsigned char* h = pieces[S.piece0 + r];
        const float* f = reinterpret_cast<const float*>(h);
        if (KIND == K_EFSIGN) { sh_sp[r] = f[0]; sh_sn[r] = -f[0]; }
        else { sh_sn[r] = f[0]; sh_sp[r] = f[1]; }
        sh_w[r] = reinterpret_cast<const uint32_t*>(h + 16);
      }
      __syncthreads();
      if (S.npieces >= 2 && S.npieces <= (uint32_t)kSignLutPieces) {
        const Divisor dv(S.divisor);
        for (uint32_t t = threadIdx.x; t < (1u << S.npieces); t += kThreads) {
          float a = 0.f;
          for (uint32_t r = 0; r < S.npieces; ++r) a = __fadd_rn(a, ((t >> r) & 1u) ? sh_sp[r] : sh_sn[r]);
          if (S.divisor != 1.0f) a = dv(a);
#pragma unroll 8
          for (int c = 0; c < 32; ++c) sh_lut[t * 32 + c] = a;
        }
        for (uint32_t i = S.npieces * kSignWords + threadIdx.x; i < kSignLutPieces * kSignWords; i += kThreads)
          sh_words[i] = 0u;   // absent pieces' rows: index bit 0
        __syncthreads();
      }
      have = false;
    }
    const uint32_t n = S.n, np = S.npieces;
    const uint32_t nwords = (n + 31) / 32;   // words a piece carries for this segment
    const uint32_t w0 = (gu - S.unit0) * kSignWords;
    const uint32_t lt = threadIdx.x * 4;      // unit-relative element of j = 0
    const uint32_t e0 = w0 * 32 + lt;
    const Divisor div(S.divisor);
    const bool ones = S.divisor == 1.0f;
    float* out = seg_out(S);
    if (np == 1) {
      const uint32_t* w = sh_w[0];
      auto comp = [](uint4& v, int c) -> uint32_t& { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; };
      uint32_t wd[kJ];
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const uint32_t e = e0 + j * kThreads * 4;
        wd[j] = have ? comp(pre[j / 4], j % 4) : (e < n ? __ldg(w + (e >> 5)) : 0u);
      }
      have = gu + 1 < u1 && sid_next == cur;   // prefetch the next unit of the segment
      if (have) {
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
          const uint32_t e = e0 + kSignUnit + j * kThreads * 4;
          comp(pre[j / 4], j % 4) = e < n ? __ldg(w + (e >> 5)) : 0u;
        }
      }
      const float sp = sh_sp[0], sn = sh_sn[0];
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const uint32_t e = e0 + j * kThreads * 4;
        const uint32_t nib = (wd[j] >> (e & 31)) & 0xFu;
        float4 v = make_float4(__fadd_rn(0.f, (nib & 1) ? sp : sn), __fadd_rn(0.f, (nib & 2) ? sp : sn),
                               __fadd_rn(0.f, (nib & 4) ? sp : sn), __fadd_rn(0.f, (nib & 8) ? sp : sn));
        if (e < n) store4_guard(out, e, n, ones ? v : div(v));
      }
      continue;
    }
    // ---- stage every piece's words of this unit in shared memory
    const uint32_t nvec = np * kSignVec;
    const bool prefetch = nvec <= (uint32_t)(kSignPre * kThreads);
    __syncthreads();   // the previous unit's words are decoded
    if (prefetch) {
      if (!have) {
#pragma unroll
        for (int m = 0; m < kSignPre; ++m) {
          const uint32_t v = threadIdx.x + m * kThreads;
          if (v < nvec) pre[m] = load_vec(v, w0, nwords);
        }
      }
#pragma unroll
      for (int m = 0; m < kSignPre; ++m) {
        const uint32_t v = threadIdx.x + m * kThreads;
        if (v < nvec) reinterpret_cast<uint4*>(sh_words)[v] = pre[m];
      }
      have = gu + 1 < u1 && sid_next == cur;   // the next unit's loads fly while this one is decoded
      if (have) {
#pragma unroll
        for (int m = 0; m < kSignPre; ++m) {
          const uint32_t v = threadIdx.x + m * kThreads;
          if (v < nvec) pre[m] = load_vec(v, w0 + kSignWords, nwords);
        }
      }
    } else {
      for (uint32_t v0 = threadIdx.x; v0 < nvec; v0 += kSignPre * kThreads) {
        uint4 t[kSignPre];
#pragma unroll
        for (int m = 0; m < kSignPre; ++m)
          if (v0 + m * kThreads < nvec) t[m] = load_vec(v0 + m * kThreads, w0, nwords);
#pragma unroll
        for (int m = 0; m < kSignPre; ++m)
          if (v0 + m * kThreads < nvec) reinterpret_cast<uint4*>(sh_words)[v0 + m * kThreads] = t[m];
      }
    }
    __syncthreads();
    if (np <= (uint32_t)kSignLutPieces) {
      // a thread decodes 8 consecutive elements (byte q of a word) per group:
      // the 8 pieces' bytes transposed into 8 index bytes (sign_index8; words
      // of pieces >= np are staged zeros), 8 lookups, one 32-byte store --
      // a warp writes 1 KB contiguous per group
      const char* lutb = reinterpret_cast<const char*>(sh_lut + lane);
      const uint32_t q = threadIdx.x & 3u;
      const bool a32 = (reinterpret_cast<uintptr_t>(out) & 31) == 0;
#pragma unroll
      for (int g = 0; g < kSignUnit / (kThreads * 8); ++g) {
        const uint32_t grp = g * kThreads + threadIdx.x;   // 8-element group of the unit
        uint32_t w[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) w[r] = sh_words[r * kSignWords + (grp >> 2)];
        uint32_t lo, hi;
        sign_index8(w, q, lo, hi);
        float v[8];   // table entry [idx][lane]: byte offset idx * 128 + lane * 4
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          v[c] = *reinterpret_cast<const float*>(lutb + (((lo >> (8 * c)) << 7) & 0x7F80u));
          v[c + 4] = *reinterpret_cast<const float*>(lutb + (((hi >> (8 * c)) << 7) & 0x7F80u));
        }
        const uint32_t e = w0 * 32 + grp * 8;
        if (a32 && e + 8 <= n) {
          st8(out + e, v);
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (e + c < n) out[e + c] = v[c];
        }
      }
      continue;
    }
    // more pieces: per float4, the pieces in rank order (the words are staged)
    for (int j = 0; j < kJ; ++j) {
      const uint32_t l = lt + j * kThreads * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t r = 0; r < np; ++r) {
        const float sp = sh_sp[r], sn = sh_sn[r];
        const uint32_t nib = (sh_words[r * kSignWords + (l >> 5)] >> (l & 31)) & 0xFu;
        acc.x = __fadd_rn(acc.x, (nib & 1) ? sp : sn);
        acc.y = __fadd_rn(acc.y, (nib & 2) ? sp : sn);
        acc.z = __fadd_rn(acc.z, (nib & 4) ? sp : sn);
        acc.w = __fadd_rn(acc.w, (nib & 8) ? sp : sn);
      }
      const uint32_t e = e0 + j * kThreads * 4;
      if (e < n) store4_guard(out, e, n, ones ? acc : div(acc));
    }
  }
}

// NONE: out = reduce(sum_r dense piece r).  Used for the sim world's
// uncompressed routines and to unpack an NCCL-reduced bucket (1 piece).
__global__ void __launch_bounds__(kThreads) h2_dense_kernel(const SegH2* __restrict__ segs,
                                                            const uint32_t* __restrict__ unit_seg,
                                                            const unsigned char* const* __restrict__ pieces) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  const uint32_t sid = unit_seg[blockIdx.x];
  const SegH2 S = segs[sid];
  const uint32_t u = blockIdx.x - S.unit0;
  const uint32_t n = S.n;
  const Divisor div(S.divisor);
  const bool ones = S.divisor == 1.0f;
  for (int j = 0; j < kUnit / (kThreads * 4); ++j) {
    const uint32_t e = u * kUnit + (j * kThreads + threadIdx.x) * 4;
    if (e >= n) break;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t r = 0; r < S.npieces; ++r) {
      const float4 v = load4_guard(reinterpret_cast<const float*>(pieces[S.piece0 + r]), e, n);
      acc.x = __fadd_rn(acc.x, v.x);
      acc.y = __fadd_rn(acc.y, v.y);
      acc.z = __fadd_rn(acc.z, v.z);
      acc.w = __fadd_rn(acc.w, v.w);
    }
    if (!ones) acc = div(acc);
    store4_guard(seg_out(S), e, n, acc);
  }
}

__global__ void __launch_bounds__(kThreads) pack_kernel(const SegH1* __restrict__ segs,
                                                        const uint32_t* __restrict__ unit_seg) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  const uint32_t sid = unit_seg[blockIdx.x];
  const SegH1 S = segs[sid];
  const uint32_t u = blockIdx.x - S.unit0;
  float* dst = reinterpret_cast<float*>(S.chunk);
  for (int j = 0; j < kUnit / (kThreads * 4); ++j) {
    const uint32_t e = u * kUnit + (j * kThreads + threadIdx.x) * 4;
    if (e >= S.n) break;
    store4_guard(dst, e, S.n, load4_stream_guard(seg_g(S), e, S.n));
  }
}

void launch_h2_sparse(const SegH2* segs, const uint32_t* tile_seg, int ntiles, const uint4* jobs, int njobs,
                      const unsigned char* const* pieces, int max_pieces, bool dense, cudaStream_t st) {
  if (ntiles == 0) return;
  if (max_pieces > 1 && dense) {
    static const int capc = [] {
      int dev = 0, sms = 148, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2_sparse_cta_kernel, kThreads, 0);
      return sms * (per_sm > 0 ? per_sm : 4);
    }();
    const int nct = (ntiles + 7) / 8;
    launch_pdl(h2_sparse_cta_kernel, nct < capc ? nct : capc, kThreads, 0, st, segs, tile_seg, (uint32_t)ntiles, pieces);
    count_launches(1);
    return;
  }
  auto cap = [](const void* fn, int smem) {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kTileThreads, smem);
    return sms * (per_sm > 0 ? per_sm : 8);
  };
  if (max_pieces <= 1) {
    // one piece: as many warps as fit, each over a contiguous tile range
    static const int cap1 = cap((const void*)h2_sparse1_kernel, 0);
    const int need = (ntiles + kTileThreads / 32 - 1) / (kTileThreads / 32);
    launch_pdl(h2_sparse1_kernel, need < cap1 ? need : cap1, kTileThreads, 0, st, segs, tile_seg, (uint32_t)ntiles,
               pieces);
    count_launches(1);
    return;
  }
  launch_pdl(h2_sparse_offsets_kernel, njobs, kThreads, 0, st, segs, jobs, pieces);
  constexpr int kSmem = kTileThreads / 32 * kTile * (int)sizeof(float);
  static const int capn = cap((const void*)h2_sparse_kernel<true>, kSmem);
  const int need = (ntiles + kTileThreads / 32 - 1) / (kTileThreads / 32);   // one warp per tile
  launch_pdl(h2_sparse_kernel<true>, need < capn ? need : capn, kTileThreads, kSmem, st, segs, tile_seg,
             (uint32_t)ntiles, pieces);
  count_launches(2);
}

void launch_h2_sign(int kind, const SegH2* segs, const uint32_t* unit_seg, int nunits,
                    const unsigned char* const* pieces, int max_pieces, cudaStream_t st) {
  if (nunits == 0) return;
  if (max_pieces < 1) max_pieces = 1;
  const int smem = (int)sign_h2_smem(max_pieces);   // words of every piece + the 32 KB table (>= 2 pieces)
  static const bool attr = [] {
    const int mx = (int)sign_h2_smem(kMaxPieces);
    return cudaFuncSetAttribute(h2_sign_kernel<K_EFSIGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) ==
               cudaSuccess &&
           cudaFuncSetAttribute(h2_sign_kernel<K_ONEBIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) ==
               cudaSuccess;
  }();
  (void)attr;
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2_sign_kernel<K_EFSIGN>, kThreads, smem);
  const int cap = sms * (per_sm > 0 ? per_sm : 4);
  const int grid = nunits < cap ? nunits : cap;
  if (kind == K_EFSIGN)
    launch_pdl(h2_sign_kernel<K_EFSIGN>, grid, kThreads, smem, st, segs, unit_seg, (uint32_t)nunits, pieces, max_pieces);
  else
    launch_pdl(h2_sign_kernel<K_ONEBIT>, grid, kThreads, smem, st, segs, unit_seg, (uint32_t)nunits, pieces, max_pieces);
  count_launches(1);
}

void launch_h2_dense(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                     const unsigned char* const* pieces, cudaStream_t st) {
  if (nunits == 0) return;
  launch_pdl(h2_dense_kernel, nunits, kThreads, 0, st, segs, unit_seg, pieces);
  count_launches(1);
}

__global__ void __launch_bounds__(kThreads) add_kernel(float* __restrict__ out, const float* __restrict__ x,
                                                      uint32_t n) {
  pdl_wait();     // predecessors in the stream are complete (PDL)
  pdl_trigger();
  for (uint32_t e = (blockIdx.x * kThreads + threadIdx.x) * 4; e < n; e += gridDim.x * kThreads * 4) {
    const float4 a = load4_guard(out, e, n), b = load4_guard(x, e, n);
    store4_guard(out, e, n, make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                                        __fadd_rn(a.w, b.w)));
  }
}

void launch_add(float* out, const float* x, uint32_t n, cudaStream_t st) {
  if (n == 0) return;
  const uint32_t blocks = std::min<uint32_t>((n + kThreads * 4 - 1) / (kThreads * 4), 148u * 8u);
  launch_pdl(add_kernel, blocks, kThreads, 0, st, out, x, n);
  count_launches(1);
}

void launch_pack(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st) {
  if (nunits == 0) return;
  launch_pdl(pack_kernel, nunits, kThreads, 0, st, segs, unit_seg);
  count_launches(1);
}

}  // namespace esp
