// EFSignSGD / Onebit h1 on sm_100a (
// EFSignSGD evaluated at P:1426, 1 bit saves "96.9%" P:791; Onebit in the
// App. D figures; error feedback P:1427).
//
// One streaming pass per step (12 B/elem + 1/8 B/elem of bits) using a LAZY
// residual: the state buffer holds last step's p and the state pair holds last
// step's scale(s), so the true residual r = fl(p - delta(p)) is recovered on
// the fly — the same fp32 operation on the same operands as an eager update,
// hence bit-identical to it.  Sign bits (p >= 0, reading R6) are packed
// LSB-first: each lane packs a nibble from its float4, 3 xor-shuffles OR the 8
// nibbles of a 32-element word, one more shuffle transposes so that each lane
// stores one word (one coalesced 128 B store per warp per 1024 elements).
// sum|p| (EFSignSGD) or the class sums/counts (Onebit) are accumulated in fp64
// and combined deterministically by the last CTA of the segment.
//
// With DECODE the input is not a gradient but the mean of npieces received
// chunks: the mid-scheme "decompress, aggregate, recompress" of quantized
// Alltoall/Allgather and Gather/Broadcast, fused.
// Both run on the persistent TMA streaming driver (stream_tma.cuh).
#include "esp_device.cuh"
#include "esp_kernels.h"
#include "stream_tma.cuh"

namespace esp {

template <int KIND>
__device__ __forceinline__ void piece_scales(const unsigned char* h, float* sp, float* sn) {
  const float* f = reinterpret_cast<const float*>(h);
  if (KIND == K_EFSIGN) {
    float s = __ldg(f);
    *sp = s;
    *sn = -s;
  } else {
    *sn = __ldg(f);
    *sp = __ldg(f + 1);
  }
}

// ---- the same h1 on the persistent TMA streaming driver (stream_tma.cuh):
// tiles of 4096 elements, 512 per warp (16 sign words per warp and tile).
// DECODE: the input is the decode-mean of S.npieces received chunks (a7, the
// mid-scheme recompression); the r stream is then the second residual r2.
template <int KIND, bool DECODE = false>
struct SignOp {
  const unsigned char* const* pieces = nullptr;
  struct State {
    float sp, sn;
    double s0, s1;
    uint32_t c0, c1;
  };
  __device__ void begin_segment(const SegH1& S, State& st, TmaHdr& h) const {
    if (DECODE) {
      // stage the segment's piece table (scales, word pointers) in shared memory
      csync<1>();
      for (uint32_t q = threadIdx.x; q < S.npieces; q += kThreads) {
        const unsigned char* p = pieces[S.piece0 + q];
        float a, b;
        piece_scales<KIND>(p, &a, &b);
        h.psp[q] = a;
        h.psn[q] = b;
        h.pw[q] = reinterpret_cast<const uint32_t*>(p + 16);
      }
      csync<1>();
    }
    st.sp = st.sn = 0.f;
    if (S.ef) {
      const float a = __ldcg(S.lazy_in), b = __ldcg(S.lazy_in + 1);
      if (KIND == K_EFSIGN) { st.sp = a; st.sn = -a; } else { st.sp = b; st.sn = a; }
    }
    st.s0 = st.s1 = 0.0;
    st.c0 = st.c1 = 0;
  }
  template <bool FULL>
  __device__ void run(const SegH1& S, const float4 (&gv)[kNJ], const float4 (&rv)[kNJ], uint32_t base,
                      State& st, TmaHdr& h, const uint32_t* sw) const {
    const uint32_t n = S.n;
    if (base >= n) return;   // warp-uniform
    const int lane = threadIdx.x & 31;
    float4 xv[kNJ];
#pragma unroll
    for (int j = 0; j < kNJ; ++j) xv[j] = gv[j];
    if (DECODE) {
      // rank-order fp32 sum of the decoded chunks from +0, then / divisor (R9);
      // the words of up to 8 pieces are loaded in one batch before any is used
#pragma unroll
      for (int j = 0; j < kNJ; ++j) xv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (uint32_t q0 = 0; q0 < S.npieces; q0 += 8) {
        const uint32_t qn = min(8u, S.npieces - q0);
        uint32_t wb[8][kNJ];
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) {
          if (q < qn) {
#pragma unroll
            for (int j = 0; j < kNJ; ++j) {
              const uint32_t e = base + j * 128 + lane * 4;
              const uint32_t l = (base & (kDgcTile - 1)) + j * 128 + lane * 4;   // tile-relative
              wb[q][j] = !(FULL || e < n) ? 0u
                         : sw             ? sw[(q0 + q) * (kDgcTile / 32) + (l >> 5)]
                                          : __ldg(h.pw[q0 + q] + (e >> 5));
            }
          }
        }
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) {
          if (q < qn) {
            const float psp = h.psp[q0 + q], psn = h.psn[q0 + q];
#pragma unroll
            for (int j = 0; j < kNJ; ++j) {
              const uint32_t e = base + j * 128 + lane * 4;
              if (FULL || e < n) {
                const uint32_t nib = (wb[q][j] >> (e & 31)) & 0xFu;
                xv[j].x = __fadd_rn(xv[j].x, (nib & 1) ? psp : psn);
                xv[j].y = __fadd_rn(xv[j].y, (nib & 2) ? psp : psn);
                xv[j].z = __fadd_rn(xv[j].z, (nib & 4) ? psp : psn);
                xv[j].w = __fadd_rn(xv[j].w, (nib & 8) ? psp : psn);
              }
            }
          }
        }
      }
      if (S.divisor != 1.0f) {
        const Divisor div(S.divisor);
#pragma unroll
        for (int j = 0; j < kNJ; ++j) xv[j] = div(xv[j]);
      }
    }
    uint32_t myword = 0;
#pragma unroll
    for (int j = 0; j < kNJ; ++j) {
      const uint32_t e = base + j * 128 + lane * 4;
      float4 p = xv[j];
      if (S.ef) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float q = f4get(rv[j], c);
          const float rt = __fsub_rn(q, q >= 0.f ? st.sp : st.sn);   // lazy residual
          f4set(p, c, __fadd_rn(f4get(xv[j], c), rt));
        }
        if (FULL) st4(S.r + e, p);
        else store4_guard(S.r, e, n, p);
      }
      uint32_t nib = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (FULL || e + c < n) {
          const float v = f4get(p, c);
          const bool b = v >= 0.f;
          nib |= (uint32_t)b << c;
          if (KIND == K_EFSIGN) {
            st.s0 += fabs((double)v);
          } else if (b) {
            st.s1 += (double)v;
            ++st.c1;
          } else {
            st.s0 += (double)v;
            ++st.c0;
          }
        }
      }
      uint32_t word = nib << (4 * (lane & 7));
      word |= __shfl_xor_sync(0xffffffffu, word, 1);
      word |= __shfl_xor_sync(0xffffffffu, word, 2);
      word |= __shfl_xor_sync(0xffffffffu, word, 4);
      const uint32_t wv = __shfl_sync(0xffffffffu, word, (lane & 3) * 8);
      if ((lane >> 2) == j) myword = wv;
    }
    uint32_t* words = reinterpret_cast<uint32_t*>(S.chunk + 16);
    if (lane < kRun / 32 && base + lane * 32 < n) words[(base >> 5) + lane] = myword;
  }
  // per (CTA, segment): the CTA's partial goes to the slot of its first unit of
  // the segment (other slots stay zero); the CTA completing the segment sums the
  // slots in unit order (deterministic for a given grid) and writes the scale(s).
  // the 4 sums of the CTA's consumer warps, in fixed order, on thread 0
  __device__ static void cta_sum4(double& a, double& b, uint32_t& ca, uint32_t& cb, TmaHdr& h) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      ca += __shfl_xor_sync(0xffffffffu, ca, o);
      cb += __shfl_xor_sync(0xffffffffu, cb, o);
    }
    csync<1>();   // previous users of h.red / h.scan are done
    if (lane == 0) {
      h.red[warp] = a;
      h.red[8 + warp] = b;
      h.scan[warp] = ca;
      h.scan[8 + warp] = cb;
    }
    csync<1>();
    if (threadIdx.x == 0) {
      a = b = 0.0;
      ca = cb = 0;
      for (int w = 0; w < kThreads / 32; ++w) {
        a += h.red[w];
        b += h.red[8 + w];
        ca += h.scan[w];
        cb += h.scan[8 + w];
      }
    }
  }
  __device__ void end_segment(const SegH1& S, uint32_t units, uint32_t first_unit, State& st, TmaHdr& h) const {
    double a = st.s0, b = st.s1;
    uint32_t ca = st.c0, cb = st.c1;
    cta_sum4(a, b, ca, cb, h);
    if (units != S.nunits) {
      // shared segment: publish this CTA's partial, the CTA completing it sums all
      if (threadIdx.x == 0) {
        S.partial[2 * first_unit] = a;
        S.partial[2 * first_unit + 1] = b;
        S.pcount[2 * first_unit] = ca;
        S.pcount[2 * first_unit + 1] = cb;
        __threadfence();
        const uint32_t old = atomicAdd(&S.st->done, units);
        h.flag = (old + units == S.nunits);
      }
      csync<1>();
      if (!h.flag) return;
      __threadfence();
      a = b = 0.0;
      ca = cb = 0;
      for (uint32_t v = threadIdx.x; v < S.nunits; v += kThreads) {
        a += __ldcg(S.partial + 2 * v);
        b += __ldcg(S.partial + 2 * v + 1);
        ca += __ldcg(S.pcount + 2 * v);
        cb += __ldcg(S.pcount + 2 * v + 1);
      }
      a = block_sum_f64<1>(a, h.red);
      b = block_sum_f64<1>(b, h.red);
      ca = block_sum_u32<1>(ca, h.scan);
      cb = block_sum_u32<1>(cb, h.scan);
    }
    // (a segment owned by one CTA is finalised directly: its sum equals the
    // slot-wise sum, which would only add exact zeros)
    if (threadIdx.x == 0) {
      float* hdr = reinterpret_cast<float*>(S.chunk);
      const uint32_t n = S.n;
      float x0, x1;
      if (KIND == K_EFSIGN) {
        x0 = n ? (float)(a / (double)n) : 0.f;   // scale = ||p||_1 / N (R7)
        x1 = 0.f;
      } else {
        x0 = ca ? (float)(a / (double)ca) : 0.f;  // mean of {p < 0} (R8)
        x1 = cb ? (float)(b / (double)cb) : 0.f;  // mean of {p >= 0}
      }
      hdr[0] = x0;
      if (KIND == K_ONEBIT) hdr[1] = x1;
      if (S.ef) {
        S.lazy_out[0] = x0;
        S.lazy_out[1] = x1;
      }
    }
    csync<1>();
  }
};

template <int KIND>
__global__ void sign_materialize_kernel(const float* __restrict__ p, const float* __restrict__ lazy,
                                        float* __restrict__ out, uint32_t n) {
  const float a = lazy[0], b = lazy[1];
  const float sp = KIND == K_EFSIGN ? a : b;
  const float sn = KIND == K_EFSIGN ? -a : a;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float q = p[i];
    out[i] = __fsub_rn(q, q >= 0.f ? sp : sn);
  }
}

int tma_stream_grid(int nunits);
int tma_stream_stages();

template <class Op>
static void launch_tma_op(const SegH1* segs, const uint32_t* unit_seg, int nunits, Op op, cudaStream_t st) {
  static bool init = [] {
    return cudaFuncSetAttribute(tma_stream_kernel<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kTmaHdrBytes + kTmaMaxStages * kTmaStageBytes)) == cudaSuccess;
  }();
  (void)init;
  const int ns = tma_stream_stages();
  tma_stream_kernel<<<tma_stream_grid(nunits), kThreads + 32, kTmaHdrBytes + ns * kTmaStageBytes, st>>>(
      segs, unit_seg, (uint32_t)nunits, ns, op);
  count_launches(1);
}

void launch_sign_h1_tma(int kind, const SegH1* segs, const uint32_t* unit_seg, int nunits,
                        const unsigned char* const* pieces, cudaStream_t st) {
  if (nunits == 0) return;
  if (kind == K_EFSIGN) {
    if (pieces) launch_tma_op(segs, unit_seg, nunits, SignOp<K_EFSIGN, true>{pieces}, st);
    else launch_tma_op(segs, unit_seg, nunits, SignOp<K_EFSIGN, false>{}, st);
  } else {
    if (pieces) launch_tma_op(segs, unit_seg, nunits, SignOp<K_ONEBIT, true>{pieces}, st);
    else launch_tma_op(segs, unit_seg, nunits, SignOp<K_ONEBIT, false>{}, st);
  }
}

void launch_sign_materialize(int kind, const float* p, const float* lazy, float* out, uint32_t n,
                             cudaStream_t st) {
  if (n == 0) return;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  if (kind == K_EFSIGN) sign_materialize_kernel<K_EFSIGN><<<blocks, 256, 0, st>>>(p, lazy, out, n);
  else sign_materialize_kernel<K_ONEBIT><<<blocks, 256, 0, st>>>(p, lazy, out, n);
  count_launches(1);
}

}  // namespace esp
