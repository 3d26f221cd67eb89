// NVLink evidence for the fused collectives' push kernel (SURVEY.md 8f
// NEXT-1): one process, 2+ GPUs; GPU 0 runs libesp's push_kernel (the same
// source, compiled in) over the jobs of an Allgather of a P-byte payload to
// every peer (one 32 KB job per chunk per destination, one arrival per job),
// timed with CUDA events; under ncu its nvltx__bytes / nvlrx__bytes give the
// bytes that crossed NVLink.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I include -o push_nvlink tools/push_nvlink.cu
//   ./push_nvlink [payload MiB]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2205_14465_b200/csrc/k_push.cu"

namespace esp {
void count_launches(int) {}
}

#define CR(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? (size_t)atoi(argv[1]) : 16;
  const size_t P = mib << 20;
  int ndev = 0;
  CR(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  const int G = ndev;
  std::vector<unsigned char*> dst(G, nullptr);
  std::vector<unsigned long long*> cnt(G, nullptr);
  for (int d = 1; d < G; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaMalloc(&dst[d], P));
    CR(cudaMalloc(&cnt[d], 8));
    CR(cudaMemset(cnt[d], 0, 8));
  }
  CR(cudaSetDevice(0));
  for (int d = 1; d < G; ++d) CR(cudaDeviceEnablePeerAccess(d, 0));
  unsigned char* src;
  CR(cudaMalloc(&src, P));
  CR(cudaMemset(src, 7, P));
  std::vector<esp::PushJob> jobs;
  for (int d = 1; d < G; ++d)
    for (size_t c = 0; c < P; c += esp::kPushChunk)
      jobs.push_back(esp::PushJob{c, c, (uint32_t)(P - c < (size_t)esp::kPushChunk ? P - c : esp::kPushChunk), (uint32_t)d});
  esp::PushJob* djobs;
  unsigned char** ddst;
  unsigned long long** dcnt;
  CR(cudaMalloc(&djobs, jobs.size() * sizeof(esp::PushJob)));
  CR(cudaMemcpy(djobs, jobs.data(), jobs.size() * sizeof(esp::PushJob), cudaMemcpyHostToDevice));
  CR(cudaMalloc(&ddst, G * sizeof(void*)));
  CR(cudaMalloc(&dcnt, G * sizeof(void*)));
  CR(cudaMemcpy(ddst, dst.data(), G * sizeof(void*), cudaMemcpyHostToDevice));
  CR(cudaMemcpy(dcnt, cnt.data(), G * sizeof(void*), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CR(cudaEventCreate(&e0));
  CR(cudaEventCreate(&e1));
  for (int rep = 0; rep < 3; ++rep) {
    CR(cudaEventRecord(e0));
    esp::launch_push(djobs, (int)jobs.size(), src, ddst, dcnt, 0);
    CR(cudaEventRecord(e1));
    CR(cudaEventSynchronize(e1));
    float ms = 0;
    CR(cudaEventElapsedTime(&ms, e0, e1));
    printf("push %zu MiB to each of %d peers: %.1f us, %.0f GB/s out of GPU 0 (%.0f GB/s per peer)\n", mib, G - 1,
           ms * 1e3, (G - 1) * P / (ms * 1e-3) / 1e9, P / (ms * 1e-3) / 1e9);
  }
  unsigned long long c = 0;
  CR(cudaSetDevice(1));
  CR(cudaMemcpy(&c, cnt[1], 8, cudaMemcpyDeviceToHost));
  unsigned char b = 0;
  CR(cudaMemcpy(&b, dst[1] + P - 1, 1, cudaMemcpyDeviceToHost));
  printf("arrivals at GPU 1: %llu (want %zu), last byte %d (want 7)\n", c, 3 * ((P + esp::kPushChunk - 1) / esp::kPushChunk),
         (int)b);
  return 0;
}
