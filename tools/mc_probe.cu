// NVLS multicast probe: does this box support switch
// multicast, and what does one multimem.st of a payload to every GPU cost
// against unicast peer stores to each?  Single process, 2+ GPUs:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_probe tools/mc_probe.cu -lcuda && ./mc_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("FAIL %s: %s\n", #x, s_); return 1; } } while (0)
#define CR(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void mc_store(float4* mc, size_t n, float base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float v = base + (float)(i & 1023);
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "f"(v), "f"(v), "f"(v),
                 "f"(v) : "memory");
  }
}
__global__ void uc_store(float4* const* dst, int ndst, size_t n, float base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float v = base + (float)(i & 1023);
    for (int d = 0; d < ndst; ++d) dst[d][i] = make_float4(v, v, v, v);
  }
}

int main() {
  CK(cuInit(0));
  int ndev = 0;
  CR(cudaGetDeviceCount(&ndev));
  printf("devices: %d\n", ndev);
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  const int G = ndev > 8 ? 8 : ndev;
  for (int d = 0; d < G; ++d) {
    int mcs = 0;
    CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
    printf("device %d multicast supported: %d\n", d, mcs);
  }
  CUmulticastObjectProp mp{};
  mp.numDevices = G;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = 64ull << 20;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (mp.size + gran - 1) / gran * gran;
  printf("granularity %zu, size %zu\n", gran, mp.size);
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < G; ++d) CK(cuMulticastAddDevice(mc, d));
  std::vector<CUmemGenericAllocationHandle> mem(G);
  std::vector<CUdeviceptr> uc(G);
  for (int d = 0; d < G; ++d) {
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CK(cuMemCreate(&mem[d], mp.size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem[d], 0, mp.size, 0));
    CK(cuMemAddressReserve(&uc[d], mp.size, gran, 0, 0));
    CK(cuMemMap(uc[d], mp.size, 0, mem[d], 0));
    CUmemAccessDesc ad{};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc[d], mp.size, &ad, 1));
  }
  CUdeviceptr mcva;
  CK(cuMemAddressReserve(&mcva, mp.size, gran, 0, 0));
  CK(cuMemMap(mcva, mp.size, 0, mc, 0));
  CUmemAccessDesc ad{};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mcva, mp.size, &ad, 1));
  // export / import round trip of the multicast handle (what a second process would do)
  int fd = -1;
  CUresult er = cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  printf("export multicast handle to fd: %d (fd %d)\n", (int)er, fd);

  CR(cudaSetDevice(0));
  const size_t n = mp.size / 16;
  cudaEvent_t e0, e1;
  CR(cudaEventCreate(&e0));
  CR(cudaEventCreate(&e1));
  mc_store<<<1184, 256>>>(reinterpret_cast<float4*>(mcva), n, 1.0f);
  CR(cudaDeviceSynchronize());
  for (int d = 0; d < G; ++d) {
    float h[4];
    CR(cudaSetDevice(d));
    CR(cudaMemcpy(h, reinterpret_cast<void*>(uc[d] + 16 * 777), 16, cudaMemcpyDeviceToHost));
    printf("device %d sees %.1f (want %.1f)\n", d, h[0], 1.0f + 777);
  }
  CR(cudaSetDevice(0));
  for (int rep = 0; rep < 2; ++rep) {
    CR(cudaEventRecord(e0));
    for (int i = 0; i < 10; ++i) mc_store<<<1184, 256>>>(reinterpret_cast<float4*>(mcva), n, 2.0f + i);
    CR(cudaEventRecord(e1));
    CR(cudaEventSynchronize(e1));
    float ms = 0;
    CR(cudaEventElapsedTime(&ms, e0, e1));
    printf("multicast store %zu MB to %d GPUs: %.1f us each, %.0f GB/s of payload\n", mp.size >> 20, G, ms * 100,
           mp.size / (ms / 10 * 1e-3) / 1e9);
  }
  // unicast: device 0 stores the same payload to every other GPU (peer access)
  std::vector<float4*> dsts;
  for (int d = 1; d < G; ++d) {
    cudaDeviceEnablePeerAccess(d, 0);
    CUmemAccessDesc a2{};
    a2.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a2.location.id = 0;
    a2.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc[d], mp.size, &a2, 1));
    dsts.push_back(reinterpret_cast<float4*>(uc[d]));
  }
  float4** ddst;
  CR(cudaMalloc(&ddst, sizeof(float4*) * dsts.size()));
  CR(cudaMemcpy(ddst, dsts.data(), sizeof(float4*) * dsts.size(), cudaMemcpyHostToDevice));
  for (int rep = 0; rep < 2; ++rep) {
    CR(cudaEventRecord(e0));
    for (int i = 0; i < 10; ++i) uc_store<<<1184, 256>>>(ddst, (int)dsts.size(), n, 3.0f + i);
    CR(cudaEventRecord(e1));
    CR(cudaEventSynchronize(e1));
    float ms = 0;
    CR(cudaEventElapsedTime(&ms, e0, e1));
    printf("unicast stores %zu MB to %d peers: %.1f us each, %.0f GB/s of payload, %.0f GB/s on the link\n",
           mp.size >> 20, (int)dsts.size(), ms * 100, mp.size / (ms / 10 * 1e-3) / 1e9,
           dsts.size() * mp.size / (ms / 10 * 1e-3) / 1e9);
  }
  printf("ok\n");
  return 0;
}
