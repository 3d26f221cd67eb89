// h2 on sm_100a: fused decompression + aggregation of the n (Allgather) or
// n^2 (Alltoall/Allgather) received pieces, written once into the gradient
// ("fuses the decompression operations"; n h2(M) and n^2 h2(M/n) of the
// cost table).
//
// Aggregation rule (reading R9): fp32 sum over pieces in rank order starting
// from +0.0f, then IEEE division by the divisor (n for MEAN).  Adding an
// implicit +0 for an absent sparse entry is the identity on a sum that started
// at +0.0f, so the sparse kernel only touches present entries.
#include "esp_device.cuh"
#include "esp_kernels.h"

namespace esp {

constexpr int kMaxPieces = 64;

// For every piece (sorted idx[kpad], 0xFFFFFFFF padding), the first entry of
// each output tile: toff[t] = lower_bound(idx, t * kTile), t = 0..ntiles.  One
// pass over the (small) pieces replaces a dependent binary search per tile.
// job = {segment, piece within segment, first entry}: kOffJob entries of one piece
__global__ void __launch_bounds__(kThreads) h2_sparse_offsets_kernel(const SegH2* __restrict__ segs,
                                                                     const uint4* __restrict__ jobs,
                                                                     const unsigned char* const* __restrict__ pieces) {
  const uint4 job = jobs[blockIdx.x];
  const SegH2 S = segs[job.x];
  const uint32_t r = job.y;
  const uint32_t ntiles = S.nunits;
  uint32_t* toff = S.toff + (size_t)r * (ntiles + 1);
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(pieces[S.piece0 + r]);
  const uint32_t iend = min(job.z + (uint32_t)kOffJob, S.kpad);
  for (uint32_t i = job.z + threadIdx.x; i < iend; i += kThreads) {
    const uint32_t v = __ldg(idx + i);
    const uint32_t t = v == 0xFFFFFFFFu ? ntiles : min(v / (uint32_t)kTile, ntiles);
    const uint32_t prev = i == 0 ? 0u : [&] {
      const uint32_t u = __ldg(idx + i - 1);
      return (u == 0xFFFFFFFFu ? ntiles : min(u / (uint32_t)kTile, ntiles)) + 1;
    }();
    for (uint32_t q = prev; q <= t; ++q) toff[q] = i;   // tiles (tile(i-1), tile(i)] start at i
    if (i == S.kpad - 1)
      for (uint32_t q = t + 1; q <= ntiles; ++q) toff[q] = S.kpad;
  }
}

// Persistent over tiles (stride gridDim.x): consecutive tiles of a CTA mostly
// belong to the same segment, so its descriptor is reloaded only on a change,
// and the next tile's offsets are fetched before this tile's work.
__global__ void __launch_bounds__(kTileThreads) h2_sparse_kernel(const SegH2* __restrict__ segs,
                                                                 const uint32_t* __restrict__ tile_seg,
                                                                 uint32_t ntiles,
                                                                 const unsigned char* const* __restrict__ pieces) {
  constexpr int kThreads = kTileThreads;   // small CTAs: many independent tiles per SM
  __shared__ __align__(16) float acc[kTile];
  __shared__ uint32_t rlo[kMaxPieces], rhi[kMaxPieces];
  uint32_t tg = blockIdx.x;
  if (tg >= ntiles) return;
  uint32_t sid = tile_seg[tg];
  SegH2 S = segs[sid];
  float* out = seg_out(S);
  uint32_t my_lo = 0, my_hi = 0;   // thread r < npieces: offsets of piece r for the current tile
  if (threadIdx.x < S.npieces) {
    const uint32_t* toff = S.toff + (size_t)threadIdx.x * (S.nunits + 1) + (tg - S.unit0);
    my_lo = __ldg(toff);
    my_hi = __ldg(toff + 1);
  }
  while (true) {
    const uint32_t t = tg - S.unit0;
    const uint32_t lo = t * kTile;
    const uint32_t hi = min(lo + (uint32_t)kTile, S.n);
    if (threadIdx.x < S.npieces) {
      rlo[threadIdx.x] = my_lo;
      rhi[threadIdx.x] = my_hi;
    }
    for (int i = threadIdx.x; i < kTile / 4; i += kThreads)
      reinterpret_cast<float4*>(acc)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    // prefetch the next tile's segment id
    const uint32_t tn = tg + gridDim.x;
    const uint32_t sid_n = tn < ntiles ? tile_seg[tn] : sid;
    __syncthreads();
    for (uint32_t r = 0; r < S.npieces; ++r) {
      const unsigned char* pc = pieces[S.piece0 + r];
      const uint32_t* idx = reinterpret_cast<const uint32_t*>(pc);
      const float* val = reinterpret_cast<const float*>(pc + 4 * (size_t)S.kpad);
      for (uint32_t i = rlo[r] + threadIdx.x; i < rhi[r]; i += kThreads) {
        const uint32_t e = __ldg(idx + i) - lo;
        acc[e] = __fadd_rn(acc[e], __ldg(val + i));   // distinct indices within a piece
      }
      __syncthreads();
    }
    const Divisor div(S.divisor);
    const bool ones = S.divisor == 1.0f;
    // next tile's offsets (same segment in the common case) before the writes
    SegH2 Sn = S;
    float* out_n = out;
    if (tn < ntiles) {
      if (sid_n != sid) {
        Sn = segs[sid_n];
        out_n = seg_out(Sn);
      }
      if (threadIdx.x < Sn.npieces) {
        const uint32_t* toff = Sn.toff + (size_t)threadIdx.x * (Sn.nunits + 1) + (tn - Sn.unit0);
        my_lo = __ldg(toff);
        my_hi = __ldg(toff + 1);
      }
    }
    for (uint32_t i = threadIdx.x * 4; lo + i < hi; i += kThreads * 4) {
      float4 v = *reinterpret_cast<const float4*>(acc + i);
      // most of a sparse tile is +0 (+0 / d = +0): divide only touched words
      if (!ones && (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f)) v = div(v);
      store4_guard(out, lo + i, S.n, v);
    }
    if (tn >= ntiles) break;
    tg = tn;
    sid = sid_n;
    S = Sn;
    out = out_n;
    __syncthreads();   // acc / rlo / rhi are reused
  }
}

template <int KIND>
__global__ void __launch_bounds__(kThreads) h2_sign_kernel(const SegH2* __restrict__ segs,
                                                           const uint32_t* __restrict__ unit_seg,
                                                           const unsigned char* const* __restrict__ pieces) {
  __shared__ float sh_sp[kMaxPieces], sh_sn[kMaxPieces];
  __shared__ const uint32_t* sh_w[kMaxPieces];
  const uint32_t sid = unit_seg[blockIdx.x];
  const SegH2 S = segs[sid];
  const uint32_t u = blockIdx.x - S.unit0;
  const uint32_t n = S.n;
  for (uint32_t r = threadIdx.x; r < S.npieces; r += kThreads) {
    const unsigned char* h = pieces[S.piece0 + r];
    const float* f = reinterpret_cast<const float*>(h);
    if (KIND == K_EFSIGN) { sh_sp[r] = f[0]; sh_sn[r] = -f[0]; }
    else { sh_sn[r] = f[0]; sh_sp[r] = f[1]; }
    sh_w[r] = reinterpret_cast<const uint32_t*>(h + 16);
  }
  __syncthreads();
  const Divisor div(S.divisor);
  const bool ones = S.divisor == 1.0f;
#pragma unroll 2
  for (int j = 0; j < kUnit / (kThreads * 4); ++j) {
    const uint32_t e = u * kUnit + (j * kThreads + threadIdx.x) * 4;
    if (e >= n) break;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t r = 0; r < S.npieces; ++r) {
      const uint32_t nib = (__ldg(sh_w[r] + (e >> 5)) >> (e & 31)) & 0xFu;
      const float sp = sh_sp[r], sn = sh_sn[r];
      acc.x = __fadd_rn(acc.x, (nib & 1) ? sp : sn);
      acc.y = __fadd_rn(acc.y, (nib & 2) ? sp : sn);
      acc.z = __fadd_rn(acc.z, (nib & 4) ? sp : sn);
      acc.w = __fadd_rn(acc.w, (nib & 8) ? sp : sn);
    }
    if (!ones) acc = div(acc);
    store4_guard(seg_out(S), e, n, acc);
  }
}

// NONE: out = reduce(sum_r dense piece r).  Used for the sim world's
// uncompressed routines and to unpack an NCCL-reduced bucket (1 piece).
__global__ void __launch_bounds__(kThreads) h2_dense_kernel(const SegH2* __restrict__ segs,
                                                            const uint32_t* __restrict__ unit_seg,
                                                            const unsigned char* const* __restrict__ pieces) {
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
                      const unsigned char* const* pieces, cudaStream_t st) {
  if (ntiles == 0) return;
  h2_sparse_offsets_kernel<<<njobs, kThreads, 0, st>>>(segs, jobs, pieces);
  static int grid_cap = [] {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h2_sparse_kernel, kTileThreads, 0);
    return sms * (per_sm > 0 ? per_sm : 8);
  }();
  const int grid = ntiles < grid_cap ? ntiles : grid_cap;
  h2_sparse_kernel<<<grid, kTileThreads, 0, st>>>(segs, tile_seg, (uint32_t)ntiles, pieces);
  count_launches(2);
}

void launch_h2_sign(int kind, const SegH2* segs, const uint32_t* unit_seg, int nunits,
                    const unsigned char* const* pieces, cudaStream_t st) {
  if (nunits == 0) return;
  if (kind == K_EFSIGN) h2_sign_kernel<K_EFSIGN><<<nunits, kThreads, 0, st>>>(segs, unit_seg, pieces);
  else h2_sign_kernel<K_ONEBIT><<<nunits, kThreads, 0, st>>>(segs, unit_seg, pieces);
  count_launches(1);
}

void launch_h2_dense(const SegH2* segs, const uint32_t* unit_seg, int nunits,
                     const unsigned char* const* pieces, cudaStream_t st) {
  if (nunits == 0) return;
  h2_dense_kernel<<<nunits, kThreads, 0, st>>>(segs, unit_seg, pieces);
  count_launches(1);
}

void launch_pack(const SegH1* segs, const uint32_t* unit_seg, int nunits, cudaStream_t st) {
  if (nunits == 0) return;
  pack_kernel<<<nunits, kThreads, 0, st>>>(segs, unit_seg);
  count_launches(1);
}

}  // namespace esp
