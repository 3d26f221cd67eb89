// Standalone experiment (not product code): achievable HBM bandwidth of the
// h1 access mix (read g, read r, write r) on B200 for
//   mode 0: persistent TMA ring, contiguous tile range per CTA (dgc_stream's layout)
//   mode 1: persistent TMA ring, chunks of `chunk` tiles dealt round-robin
//   mode 2: plain grid-stride float4 LDG/STG
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2205_14465_b200/csrc \
//        tools/stream_bench.cu -o gpurun_out/stream_bench
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "esp_device.cuh"

using namespace esp;
constexpr int kT = 4096;           // floats per tile
constexpr int kStages = 4;
constexpr int kStage = 2 * kT * 4;  // g + r

__global__ void __launch_bounds__(288, 1) tma_add(const float* g, float* r, uint32_t ntiles, int mode, int chunk) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[kStages], empty[kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // tile sequence of this CTA
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t c0 = (uint32_t)((uint64_t)b * ntiles / G), c1 = (uint32_t)((uint64_t)(b + 1) * ntiles / G);
  auto tile_at = [&](uint32_t i, uint32_t* t) -> bool {
    if (mode == 0) {
      *t = c0 + i;
      return *t < c1;
    }
    const uint32_t ch = i / chunk, w = i % chunk;
    *t = (ch * G + b) * chunk + w;
    return *t < ntiles;
  };
  if (warp == 8) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      bool wrapped = false;
      uint32_t t;
      for (uint32_t i = 0; tile_at(i, &t); ++i) {
        if (wrapped) mbar_wait(&empty[stage], phase ^ 1);
        float* sg = reinterpret_cast<float*>(smem + stage * kStage);
        mbar_arrive_expect_tx(&full[stage], 2 * kT * 4);
        tma_load_1d(sg, g + (size_t)t * kT, kT * 4, &full[stage], pol);
        tma_load_1d(sg + kT, r + (size_t)t * kT, kT * 4, &full[stage], pol);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
          wrapped = true;
        }
      }
    }
    return;
  }
  int stage = 0;
  uint32_t phase = 0;
  uint32_t t;
  for (uint32_t i = 0; tile_at(i, &t); ++i) {
    mbar_wait(&full[stage], phase);
    const float* sg = reinterpret_cast<const float*>(smem + stage * kStage) + warp * 512 + lane * 4;
    float4 av[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 a = lds4(sg + j * 128), c = lds4(sg + kT + j * 128);
      av[j] = make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1;
    }
    float* rp = r + (size_t)t * kT + warp * 512 + lane * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) st4(rp + j * 128, av[j]);
  }
}

__global__ void plain_add(const float4* g, float4* r, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = g[i], c = r[i];
    r[i] = make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w);
  }
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 336226304ull;   // BERT-large, whole tiles
  const uint32_t ntiles = (uint32_t)(n / kT);
  float *g, *r;
  cudaMalloc(&g, n * 4);
  cudaMalloc(&r, n * 4);
  cudaMemset(g, 0, n * 4);
  cudaMemset(r, 0, n * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_add, cudaFuncAttributeMaxDynamicSharedMemorySize, kStages * kStage);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn) {
    float best = 1e9f;
    for (int it = 0; it < 12; ++it) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2 && ms < best) best = ms;
    }
    const double bytes = 12.0 * (double)ntiles * kT;
    printf("%-28s %8.1f us  %6.3f TB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  };
  run("tma contiguous", [&] { tma_add<<<sms, 288, kStages * kStage>>>(g, r, ntiles, 0, 1); });
  for (int ch : {1, 4, 16, 64})
    run((std::string("tma chunk ") + std::to_string(ch)).c_str(),
        [&] { tma_add<<<sms, 288, kStages * kStage>>>(g, r, ntiles, 1, ch); });
  for (int per : {4, 8, 16})
    run((std::string("plain grid ") + std::to_string(per) + "/SM").c_str(),
        [&] { plain_add<<<sms * per, 256>>>((const float4*)g, (float4*)r, (size_t)ntiles * kT / 4); });
  return 0;
}
