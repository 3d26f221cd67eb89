// Persistent warp-specialised streaming driver for the h1 passes (sm_100a):
// one producer warp streams tiles of g (and r when error feedback is on) into
// an `ns`-stage shared-memory ring with 1D TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx); 8 consumer warps each take one 512-element run of a
// tile into registers, release the stage, and hand the run to an operation
// (`Op`) that writes the compressed output and the EF state.  Every CTA owns a
// contiguous range of the bucket's tile table, so it mostly stays inside one
// segment; Op::end_segment is called once per (CTA, segment) for
// per-segment bookkeeping.  Segments that are not 16-byte aligned (sim worlds
// with odd tensor sizes) or tails that are not a multiple of 16 bytes are
// read with guarded LDG instead.
#pragma once
#include "esp_device.cuh"

namespace esp {

constexpr int kTmaMaxStages = 6;
struct TmaHdr {
  uint64_t full[kTmaMaxStages], empty[kTmaMaxStages];
  double red[16];
  uint32_t scan[280];
  uint32_t misc[8];
  int flag;
};
constexpr size_t kTmaHdrBytes = (sizeof(TmaHdr) + 127) / 128 * 128;
constexpr size_t kTmaStageBytes = 2 * kDgcTile * sizeof(float);
__device__ __forceinline__ float* tma_stage_g(unsigned char* smem, int s) {
  return reinterpret_cast<float*>(smem + kTmaHdrBytes + (size_t)s * kTmaStageBytes);
}
__device__ __forceinline__ float* tma_stage_r(unsigned char* smem, int s) { return tma_stage_g(smem, s) + kDgcTile; }

template <class Op>
__global__ void __launch_bounds__(kThreads + 32, 1)
    tma_stream_kernel(const SegH1* __restrict__ segs, const uint32_t* __restrict__ unit_seg, uint32_t nunits,
                      int ns, Op op) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TmaHdr& hdr = *reinterpret_cast<TmaHdr*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t u0 = (uint32_t)((uint64_t)blockIdx.x * nunits / gridDim.x);
  const uint32_t u1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * nunits / gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&hdr.full[s], 1);
      mbar_init(&hdr.empty[s], kThreads / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kThreads / 32) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      uint32_t cur = 0xFFFFFFFFu, unit0 = 0, n = 0;
      const float* gseg = nullptr;
      const float* rseg = nullptr;
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
          ef = S.ef != 0;
        }
        if (wrapped) mbar_wait(&hdr.empty[stage], phase ^ 1);
        const uint32_t start = (u - unit0) * kDgcTile;
        const uint32_t len = min((uint32_t)kDgcTile, n - start);
        const float* g = gseg + start;
        const float* r = rseg + start;
        const uint32_t bytes = (len * 4) & ~15u;
        if (bytes && al16(g) && (!ef || al16(r))) {
          mbar_arrive_expect_tx(&hdr.full[stage], bytes * (ef ? 2 : 1));
          tma_load_1d(tma_stage_g(smem_raw, stage), g, bytes, &hdr.full[stage], pol);
          if (ef) tma_load_1d(tma_stage_r(smem_raw, stage), r, bytes, &hdr.full[stage], pol);
        } else {
          mbar_arrive(&hdr.full[stage]);
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

  typename Op::State st;
  uint32_t cur = 0xFFFFFFFFu, cur_units = 0, first_unit = 0;
  const float* g = nullptr;
  SegH1 S{};
  uint32_t sid_next = u0 < u1 ? unit_seg[u0] : 0u;
  int stage = 0;
  uint32_t phase = 0;
  for (uint32_t u = u0; u < u1; ++u) {
    const uint32_t sid = sid_next;
    if (u + 1 < u1) sid_next = unit_seg[u + 1];
    if (sid != cur) {
      if (cur != 0xFFFFFFFFu) op.end_segment(S, cur_units, first_unit, st, hdr);
      cur = sid;
      S = segs[sid];
      g = seg_g(S);
      cur_units = 0;
      first_unit = u - S.unit0;
      op.begin_segment(S, st);
    }
    ++cur_units;
    const uint32_t start = (u - S.unit0) * kDgcTile;
    const uint32_t n = S.n;
    const uint32_t len = min((uint32_t)kDgcTile, n - start);
    const uint32_t bytes = (len * 4) & ~15u;
    const bool tma = bytes && al16(g + start) && (!S.ef || al16(S.r + start));
    mbar_wait(&hdr.full[stage], phase);
    const uint32_t lbase = warp * kRun;
    const uint32_t base = start + lbase;
    const bool full = tma && start + kDgcTile <= n;   // whole tile staged, no bounds
    float4 gv[kNJ], rv[kNJ];
    if (full) {
      const float* sg = tma_stage_g(smem_raw, stage) + lbase + lane * 4;
      const float* sr = tma_stage_r(smem_raw, stage) + lbase + lane * 4;
#pragma unroll
      for (int j = 0; j < kNJ; ++j) {
        gv[j] = lds4(sg + j * 128);
        rv[j] = S.ef ? lds4(sr + j * 128) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kNJ; ++j) {
        const uint32_t l = lbase + j * 128 + lane * 4;
        if (tma && l + 4 <= bytes / 4) {
          gv[j] = lds4(tma_stage_g(smem_raw, stage) + l);
          rv[j] = S.ef ? lds4(tma_stage_r(smem_raw, stage) + l) : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          gv[j] = load4_guard(g, start + l, n);
          rv[j] = S.ef ? load4_guard(S.r, start + l, n) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&hdr.empty[stage]);
    if (++stage == ns) {
      stage = 0;
      phase ^= 1;
    }
    if (full) op.template run<true>(S, gv, rv, base, st);
    else op.template run<false>(S, gv, rv, base, st);
  }
  if (cur != 0xFFFFFFFFu) op.end_segment(S, cur_units, first_unit, st, hdr);
}

}  // namespace esp
