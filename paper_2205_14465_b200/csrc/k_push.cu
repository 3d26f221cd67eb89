// Push kernel of the fused collectives: the
// producer (DGC write, sign h1 / a7) has written its payload to local HBM; this
// kernel moves it into the receiving ranks' buffers over NVLink 5 peer memory
// (CUDA IPC mappings of their plan arenas) and signals each arrival.  It
// replaces ncclAllGather / ncclAlltoAll / ncclGather / ncclBroadcast for the
// byte-moving routines of the cost table: every chunk is stored once,
// directly at its final place on every rank that reads it.
//
// One CTA per job of <= kPushChunk bytes: 8 x 16 B loads in flight per thread,
// then 8 x 16 B peer stores, repeated; the CTA barrier orders the block's stores before
// thread 0's system-scope fence (cumulative), which precedes the arrival
// increment on the destination rank's counter.
#include "esp_device.cuh"
#include "esp_kernels.h"

namespace esp {

// 64 threads per CTA (about 3K registers): push CTAs fit next to a persistent
// streaming kernel (1 CTA/SM, most of the register file) of the next bucket,
// so the exchange of bucket b overlaps h1 of bucket b + 1
constexpr int kPushThreads = 64;
__global__ void __launch_bounds__(kPushThreads) push_kernel(const PushJob* __restrict__ jobs,
                                                            const unsigned char* __restrict__ src,
                                                            unsigned char* const* __restrict__ dsts,
                                                            unsigned long long* const* __restrict__ cnts) {
  const PushJob J = jobs[blockIdx.x];
  const uint4* s = reinterpret_cast<const uint4*>(src + J.src_off);
  uint4* d = reinterpret_cast<uint4*>(dsts[J.d] + J.dst_off);
  const uint32_t nv = J.bytes / 16;
  constexpr int kV = 8;   // 16 B loads in flight per thread
  for (uint32_t e0 = 0; e0 < nv; e0 += kV * kPushThreads) {
    uint4 v[kV];
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const uint32_t e = e0 + i * kPushThreads + threadIdx.x;
      if (e < nv) v[i] = __ldcg(s + e);
    }
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const uint32_t e = e0 + i * kPushThreads + threadIdx.x;
      if (e < nv) d[e] = v[i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    atomicAdd_system(cnts[J.d], 1ull);
  }
}

// Multicast variant (NVLS, mcast.cu): every job's bytes are stored ONCE to
// the multicast alias of the destination slot (the NVSwitch writes them into
// every rank's copy), then one system-scope release + multicast reduction
// bumps every rank's arrival counter at once.
__global__ void __launch_bounds__(kPushThreads) push_mc_kernel(const PushJob* __restrict__ jobs,
                                                               const unsigned char* __restrict__ src,
                                                               unsigned char* mc_dst, unsigned long long* mc_cnt) {
  const PushJob J = jobs[blockIdx.x];
  const uint4* s = reinterpret_cast<const uint4*>(src + J.src_off);
  unsigned char* d = mc_dst + J.dst_off;
  const uint32_t nv = J.bytes / 16;
  constexpr int kV = 8;
  for (uint32_t e0 = 0; e0 < nv; e0 += kV * kPushThreads) {
    uint4 v[kV];
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const uint32_t e = e0 + i * kPushThreads + threadIdx.x;
      if (e < nv) v[i] = __ldcg(s + e);
    }
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const uint32_t e = e0 + i * kPushThreads + threadIdx.x;
      if (e < nv)   // a 128-bit store to the multicast alias (bits move unchanged)
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(d + 16ull * e),
                     "f"(__uint_as_float(v[i].x)), "f"(__uint_as_float(v[i].y)), "f"(__uint_as_float(v[i].z)),
                     "f"(__uint_as_float(v[i].w))
                     : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc_cnt), "l"(1ull) : "memory");
  }
}

void launch_push_mc(const PushJob* jobs, int njobs, const unsigned char* src, unsigned char* mc_dst,
                    unsigned long long* mc_cnt, cudaStream_t st) {
  if (njobs == 0) return;
  push_mc_kernel<<<njobs, kPushThreads, 0, st>>>(jobs, src, mc_dst, mc_cnt);
  count_launches(1);
}

void launch_push(const PushJob* jobs, int njobs, const unsigned char* src, unsigned char* const* dsts,
                 unsigned long long* const* cnts, cudaStream_t st) {
  if (njobs == 0) return;
  push_kernel<<<njobs, kPushThreads, 0, st>>>(jobs, src, dsts, cnts);
  count_launches(1);
}

}  // namespace esp
