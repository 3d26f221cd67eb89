// Persistent warp-specialised streaming driver for the h1 passes (sm_100a):
// one producer warp streams tiles of g (and r when error feedback is on) into
// an `ns`-stage shared-memory ring with 1D TMA bulk copies (cp.async.bulk +
// mbarrier complete_tx); 8 consumer warps each take one 512-element run of a
// tile into registers, release the stage, and hand the run to an operation
// (`Op`) that writes the compressed output and the EF state.  Several groups
// of 8 consumer warps per CTA (see tma_stream_kernel).  Every CTA owns a
// contiguous range of the bucket's tile table, so it mostly stays inside one
// segment; Op::end_segment is called once per (CTA, segment) for
// per-segment bookkeeping.  Segments that are not 16-byte aligned (sim worlds
// with odd tensor sizes) or tails that are not a multiple of 16 bytes are
// read with guarded LDG instead.
#pragma once
#include <cstdlib>
#include "esp_device.cuh"
#include "esp_kernels.h"

namespace esp {

constexpr int kTmaMaxStages = 6;
constexpr int kMaxPiecesTma = 64;
constexpr int kTmaGroups = 3;   // max consumer groups of 8 warps (Op::kGroups <= this)
// per consumer group: reduction scratch and the op's per-segment tables
struct TmaGroup {
  double red[16];
  uint32_t scan[280];
  uint32_t misc[8];
  int flag;
  // per-warp scratch of ops that address a run's elements by position (Randomk)
  alignas(16) float wscr[kThreads / 32][kRun];
  uint32_t wsel[kThreads / 32][kRun / 32];
};
struct TmaHdr {
  uint64_t full[kTmaMaxStages], empty[kTmaMaxStages];
  TmaGroup grp[kTmaGroups];
};
constexpr size_t kTmaHdrBytes = (sizeof(TmaHdr) + 127) / 128 * 128;
constexpr size_t kTmaStageBytes = 2 * kDgcTile * sizeof(float);
__device__ __forceinline__ float* tma_stage_g(unsigned char* smem, int s) {
  return reinterpret_cast<float*>(smem + kTmaHdrBytes + (size_t)s * kTmaStageBytes);
}
__device__ __forceinline__ float* tma_stage_r(unsigned char* smem, int s) { return tma_stage_g(smem, s) + kDgcTile; }

// NCG consumer groups: group c takes the CTA's tiles c, c + NCG, ... (stage
// i mod ns, ns a multiple of NCG so that a group's uses of a stage are
// consecutive phases of it); group c synchronises on named barrier 1 + c and
// owns hdr.grp[c].  Op's segment hooks are templated on that barrier id.
template <class Op, int NCG>
__global__ void __launch_bounds__(NCG * kThreads + 32, 1)
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
  pdl_wait();   // the prologue above overlapped the predecessor's tail (PDL)
  pdl_trigger();

  if (warp == NCG * kThreads / 32) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      uint32_t cur = 0xFFFFFFFFu, unit0 = 0, n = 0;
      const float* gseg = nullptr;
      const float* rseg = nullptr;
      bool ef = false;
      uint32_t npieces = 0, piece0 = 0;
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
          gseg = S.gptr ? seg_g(S) : nullptr;   // a7 segments have no g stream
          rseg = S.r;
          ef = S.ef != 0;
          // decoding segments (a7): the tile's sign words of every piece are
          // staged in the (unused) g slot, kDgcTile/32 words per piece
          npieces = (!gseg && op.pieces && op.stage_words) ? S.npieces : 0u;
          piece0 = S.piece0;
        }
        if (wrapped) mbar_wait(&hdr.empty[stage], phase ^ 1);
        const uint32_t start = (u - unit0) * kDgcTile;
        const uint32_t len = min((uint32_t)kDgcTile, n - start);
        const float* g = gseg + start;
        const float* r = rseg + start;
        const uint32_t bytes = (len * 4) & ~15u;
        const uint32_t wbytes = (((len + 31) / 32) * 4 + 15) & ~15u;
        const uint32_t nstreams = (gseg ? 1u : 0u) + (ef ? 1u : 0u);
        if (bytes && (nstreams || npieces) && (!gseg || al16(g)) && (!ef || al16(r))) {
          mbar_arrive_expect_tx(&hdr.full[stage], bytes * nstreams + wbytes * npieces);
          if (gseg) tma_load_1d(tma_stage_g(smem_raw, stage), g, bytes, &hdr.full[stage], pol);
          if (ef) tma_load_1d(tma_stage_r(smem_raw, stage), r, bytes, &hdr.full[stage], pol);
          for (uint32_t q = 0; q < npieces; ++q)
            tma_load_1d(tma_stage_g(smem_raw, stage) + q * (kDgcTile / 32),
                        op.pieces[piece0 + q] + 16 + start / 8, wbytes, &hdr.full[stage], pol);
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

  const int cg = NCG == 1 ? 0 : warp / (kThreads / 32);
  TmaGroup& gh = hdr.grp[cg];
  auto begin_seg = [&](const SegH1& S, typename Op::State& st) {
    if (NCG == 1 || cg == 0) op.template begin_segment<1>(S, st, gh);
    else if (cg == 1) op.template begin_segment<2>(S, st, gh);
    else op.template begin_segment<3>(S, st, gh);
  };
  auto end_seg = [&](const SegH1& S, uint32_t units, uint32_t first, typename Op::State& st) {
    if (NCG == 1 || cg == 0) op.template end_segment<1>(S, units, first, st, gh);
    else if (cg == 1) op.template end_segment<2>(S, units, first, st, gh);
    else op.template end_segment<3>(S, units, first, st, gh);
  };
  typename Op::State st;
  uint32_t cur = 0xFFFFFFFFu, cur_units = 0, first_unit = 0;
  const float* g = nullptr;
  SegH1 S{};
  uint32_t sid_next = u0 + cg < u1 ? unit_seg[u0 + cg] : 0u;
  int stage = cg;
  uint32_t phase = 0;
  for (uint32_t u = u0 + cg; u < u1; u += NCG) {
    const uint32_t sid = sid_next;
    if (u + NCG < u1) sid_next = unit_seg[u + NCG];
    if (sid != cur) {
      if (cur != 0xFFFFFFFFu) end_seg(S, cur_units, first_unit, st);
      cur = sid;
      S = segs[sid];
      g = S.gptr ? seg_g(S) : nullptr;
      cur_units = 0;
      first_unit = u - S.unit0;
      begin_seg(S, st);
    }
    ++cur_units;
    const uint32_t start = (u - S.unit0) * kDgcTile;
    const uint32_t n = S.n;
    const uint32_t len = min((uint32_t)kDgcTile, n - start);
    const uint32_t bytes = (len * 4) & ~15u;
    const bool has_g = g != nullptr;
    const bool dec = !has_g && op.pieces && S.npieces > 0;
    const bool staged = dec && op.stage_words;   // the pieces' words ride in the g slot
    const bool tma = bytes && (has_g || S.ef || staged) && (!has_g || al16(g + start)) && (!S.ef || al16(S.r + start));
    mbar_wait(&hdr.full[stage], phase);
    const uint32_t lbase = (warp & 7) * kRun;
    const uint32_t base = start + lbase;
    const bool full = tma && start + kDgcTile <= n;   // whole tile staged, no bounds
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 gv[kNJ], rv[kNJ];
    if (full) {
      const float* sg = tma_stage_g(smem_raw, stage) + lbase + lane * 4;
      const float* sr = tma_stage_r(smem_raw, stage) + lbase + lane * 4;
#pragma unroll
      for (int j = 0; j < kNJ; ++j) {
        gv[j] = has_g ? lds4(sg + j * 128) : zero4;
        rv[j] = S.ef ? lds4(sr + j * 128) : zero4;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kNJ; ++j) {
        const uint32_t l = lbase + j * 128 + lane * 4;
        if (tma && l + 4 <= bytes / 4) {
          gv[j] = has_g ? lds4(tma_stage_g(smem_raw, stage) + l) : zero4;
          rv[j] = S.ef ? lds4(tma_stage_r(smem_raw, stage) + l) : zero4;
        } else {
          gv[j] = has_g ? load4_guard(g, start + l, n) : zero4;
          rv[j] = S.ef ? load4_guard(S.r, start + l, n) : zero4;
        }
      }
    }
    // staged sign words of a decoding op are read inside run: release after it
    const uint32_t* sw = (tma && staged) ? reinterpret_cast<const uint32_t*>(tma_stage_g(smem_raw, stage)) : nullptr;
    const int used = stage;
    if (!sw) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&hdr.empty[used]);
    }
    stage += NCG;
    if (stage >= ns) {
      stage -= ns;
      phase ^= 1;
    }
    if (full) op.template run<true>(S, gv, rv, base, st, gh, sw);
    else op.template run<false>(S, gv, rv, base, st, gh, sw);
    if (sw) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&hdr.empty[used]);
    }
  }
  if (cur != 0xFFFFFFFFu) end_seg(S, cur_units, first_unit, st);
}

int tma_stream_grid(int nunits);
int tma_stream_stages();

// host: launch the driver for Op over a bucket's tile table (one CTA per SM)
// with NCG consumer groups
template <class Op, int NCG>
static void launch_tma_op_n(const SegH1* segs, const uint32_t* unit_seg, int nunits, Op op, cudaStream_t st) {
  // stages: what fits next to the header in 227 KB, a multiple of the group count
  constexpr int kFit = (int)((227 * 1024 - kTmaHdrBytes) / kTmaStageBytes);
  constexpr int kMaxNs = (kFit < kTmaMaxStages ? kFit : kTmaMaxStages) / NCG * NCG;
  static_assert(kMaxNs >= NCG, "one stage per consumer group at least");
  static bool init = [] {
    return cudaFuncSetAttribute(tma_stream_kernel<Op, NCG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kTmaHdrBytes + kMaxNs * kTmaStageBytes)) == cudaSuccess;
  }();
  (void)init;
  int ns = tma_stream_stages();
  ns = ns < NCG ? NCG : (ns > kMaxNs ? kMaxNs : ns - ns % NCG);
  launch_pdl(tma_stream_kernel<Op, NCG>, tma_stream_grid(nunits), NCG * kThreads + 32,
             kTmaHdrBytes + ns * kTmaStageBytes, st, segs, unit_seg, (uint32_t)nunits, ns, op);
  count_launches(1);
}

// Op::kGroups consumer groups of 8 warps
template <class Op>
static void launch_tma_op(const SegH1* segs, const uint32_t* unit_seg, int nunits, Op op, cudaStream_t st) {
  launch_tma_op_n<Op, Op::kGroups>(segs, unit_seg, nunits, op, st);
}

}  // namespace esp
