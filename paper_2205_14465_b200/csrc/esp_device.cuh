// Device helpers shared by the sm_100a kernels of this library.
// (The CPU oracle under oracle/ shares none of this.)
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

#include "esp_tables.h"

namespace esp {

__device__ __forceinline__ uint32_t fkey(float x) {
  // |x| as an order-preserving unsigned key (reading R2)
  return __float_as_uint(x) & 0x7FFFFFFFu;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// Streaming (read-once) 128-bit load: do not allocate in L1.
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ float4 ld4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

__device__ __forceinline__ void st4(float* p, float4 v) {
  *reinterpret_cast<float4*>(p) = v;
}

__device__ __forceinline__ float f4get(const float4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}
__device__ __forceinline__ void f4set(float4& v, int c, float x) {
  if (c == 0) v.x = x; else if (c == 1) v.y = x; else if (c == 2) v.z = x; else v.w = x;
}

__device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Load 4 consecutive floats at element e of an n-element array; out-of-range -> 0.
// Segments of a sim world may start at any float offset: the vector path is
// taken only when the address is 16-byte aligned.
__device__ __forceinline__ float4 load4_guard(const float* base, uint32_t e, uint32_t n) {
  if (e + 3 < n && al16(base + e)) return ld4(base + e);
  if (e + 3 < n) return make_float4(base[e], base[e + 1], base[e + 2], base[e + 3]);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e < n) v.x = base[e];
  if (e + 1 < n) v.y = base[e + 1];
  if (e + 2 < n) v.z = base[e + 2];
  return v;
}
__device__ __forceinline__ float4 load4_stream_guard(const float* base, uint32_t e, uint32_t n) {
  if (e + 3 < n && al16(base + e)) return ld_stream4(base + e);
  if (e + 3 < n) return make_float4(base[e], base[e + 1], base[e + 2], base[e + 3]);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e < n) v.x = base[e];
  if (e + 1 < n) v.y = base[e + 1];
  if (e + 2 < n) v.z = base[e + 2];
  return v;
}
__device__ __forceinline__ void store4_guard(float* base, uint32_t e, uint32_t n, float4 v) {
  if (e + 3 < n && al16(base + e)) { st4(base + e, v); return; }
  if (e + 3 < n) { base[e] = v.x; base[e + 1] = v.y; base[e + 2] = v.z; base[e + 3] = v.w; return; }
  if (e < n) base[e] = v.x;
  if (e + 1 < n) base[e + 1] = v.y;
  if (e + 2 < n) base[e + 2] = v.z;
}

// x / d for the aggregation divisor d (reading R9: IEEE division).  For a
// power-of-two d the product with the exact reciprocal is the same correctly
// rounded value (also for subnormal results), at a fraction of the cost; n =
// 1, 2, 4, 8 ranks are all powers of two.
struct Divisor {
  float d, rcp;
  bool pow2;
  __device__ __forceinline__ explicit Divisor(float dd) : d(dd) {
    const uint32_t b = __float_as_uint(dd);
    pow2 = (b & 0x007FFFFFu) == 0 && ((b >> 23) & 0xFF) > 0 && ((b >> 23) & 0xFF) < 254;
    rcp = pow2 ? __uint_as_float((uint32_t)(254 - ((b >> 23) & 0xFF)) << 23) : 0.f;
  }
  __device__ __forceinline__ float operator()(float x) const { return pow2 ? __fmul_rn(x, rcp) : __fdiv_rn(x, d); }
  __device__ __forceinline__ float4 operator()(float4 v) const {
    return make_float4((*this)(v.x), (*this)(v.y), (*this)(v.z), (*this)(v.w));
  }
};

// ---- CTA-wide scans / reductions for 256 threads ---------------------------------
// BAR = 0: __syncthreads; BAR > 0: named barrier BAR over the first 256 threads
// (the consumer warps of a warp-specialised kernel).
// BAR = b > 0 also serves the b-th group of 256 consumer threads (threads
// 256(b-1) .. 256b-1) of a kernel with several consumer groups.
template <int BAR>
__device__ __forceinline__ void csync() {
  if (BAR == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(kThreads) : "memory");
}
// thread index within the 256 threads that take part in barrier BAR
template <int BAR>
__device__ __forceinline__ int ctid() {
  return BAR == 0 ? (int)threadIdx.x : (int)(threadIdx.x & (kThreads - 1));
}

// Exclusive scan of v over the CTA in thread order.  `sh` needs 9 uint32.
template <int BAR = 0>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total, uint32_t* sh) {
  const int lane = threadIdx.x & 31, warp = ctid<BAR>() >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  csync<BAR>();
  if (warp == 0) {
    uint32_t w = lane < (kThreads / 32) ? sh[lane] : 0u;
    uint32_t s = w;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < 8) sh[lane] = s - w;
    if (lane == 7) sh[8] = s;
  }
  csync<BAR>();
  uint32_t r = x - v + sh[warp];
  *total = sh[8];
  csync<BAR>();
  return r;
}

template <int BAR = 0>
__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v, uint32_t* sh) {
  uint32_t t;
  block_excl_scan<BAR>(v, &t, sh);
  return t;
}

// Deterministic fp64 CTA sum (fixed shuffle tree then warp order).  sh: 8 doubles.
template <int BAR = 0>
__device__ __forceinline__ double block_sum_f64(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = ctid<BAR>() >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[warp] = v;
  csync<BAR>();
  double t = 0.0;
  if (ctid<BAR>() == 0) {
    for (int w = 0; w < kThreads / 32; ++w) t += sh[w];
    sh[0] = t;
  }
  csync<BAR>();
  t = sh[0];
  csync<BAR>();
  return t;
}

// ---- named barrier among the first `nthreads` threads (consumer warps of a
// warp-specialised CTA; the producer warp never joins)
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- mbarrier + 1D TMA bulk copy (cp.async.bulk, SASS UBLKCP) ------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy; completes `bytes` of transaction count on `bar`.
// src, dst 16-byte aligned, bytes a multiple of 16.  L2 evict-first: read once.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// shared -> global bulk store (bulk-group completion); src/dst 16-byte aligned
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
               "cp.async.bulk.commit_group;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// wait until every committed bulk store of this thread has READ its smem source
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// make this thread's generic-proxy smem writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// "Last CTA of a segment" election: every CTA calls this after its global
// writes; returns true in exactly one CTA (the last to arrive).
__device__ __forceinline__ bool last_cta(uint32_t* counter, uint32_t expected, int* sh_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t old = atomicAdd(counter, 1u);
    *sh_flag = (old == expected - 1);
  }
  __syncthreads();
  bool last = *sh_flag != 0;
  if (last) __threadfence();
  return last;
}

// ---- sign decode through a lookup table ------------------------------------------
// With np <= 8 pieces an element's decoded rank-order sum depends only on its
// np sign bits: lut[t] = (((+0 + x_0(t)) + x_1(t)) + ...) / divisor with
// x_r(t) = bit r of t ? pos_r : neg_r -- the same fp32 operations in the same
// order as the sequential decode, so bit-identical to it.  The np bits of 4
// consecutive elements are gathered as 4 index bytes: spread4(nib) moves bit c
// of a nibble to bit 8c (the partial products of nib * 0x204081 do not
// overlap), shifted to bit r for piece r.
constexpr int kSignLutPieces = 8;
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// The 8 index bytes of 8 consecutive elements at once: byte q of each of the
// 8 pieces' words (zero words for absent pieces) gathered into a 64-bit 8x8
// bit matrix M[r][e] = piece r's bit of element e (byte r = lo/hi byte r & 3),
// transposed in registers (three delta swaps) so that byte e holds element e's
// np bits = its table index.  ~27 integer ops per 8 elements instead of 4 per
// piece and element.
__device__ __forceinline__ void sign_index8(const uint32_t (&w)[8], uint32_t q, uint32_t& lo, uint32_t& hi) {
  const uint32_t sel = q | ((q + 4u) << 4);   // [a.q, b.q]
  lo = __byte_perm(__byte_perm(w[0], w[1], sel), __byte_perm(w[2], w[3], sel), 0x5410);
  hi = __byte_perm(__byte_perm(w[4], w[5], sel), __byte_perm(w[6], w[7], sel), 0x5410);
  uint32_t t;
  t = (lo ^ (lo >> 7)) & 0x00AA00AAu; lo ^= t ^ (t << 7);
  t = (hi ^ (hi >> 7)) & 0x00AA00AAu; hi ^= t ^ (t << 7);
  t = (lo ^ (lo >> 14)) & 0x0000CCCCu; lo ^= t ^ (t << 14);
  t = (hi ^ (hi >> 14)) & 0x0000CCCCu; hi ^= t ^ (t << 14);
  t = (lo ^ (hi << 4)) & 0xF0F0F0F0u; lo ^= t; hi ^= t >> 4;
}

// one 32-byte store (STG.256 on sm_100) of 8 consecutive floats; p 32-byte aligned
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

// ---- programmatic dependent launch (PDL) ------------------------------------------
// The kernels of a call form one chain on the caller's stream (sample ->
// stream -> fallback -> refine -> write -> h2 ...).  Each is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (launch_pdl), so its
// CTAs are scheduled while its predecessor drains instead of after it:
// pdl_trigger() lets the successor launch; pdl_wait() (griddepcontrol.wait)
// blocks until every predecessor grid has completed and its memory is
// visible.  EVERY kernel launched with launch_pdl calls pdl_wait() before it
// touches memory a predecessor writes (static tables may be read before).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace esp
