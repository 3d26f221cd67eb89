// NVLS multicast regions (mcast.cu): one multicast object per plan whose
// memory every rank maps twice (its own copy; the team-wide multicast alias).
#pragma once
#include <cuda.h>
#include <cstddef>
#include <cstdint>

struct esp_world_s;

namespace esp {

struct McRegion {
  CUmemGenericAllocationHandle mc = 0, phys = 0;
  bool have_mc = false, have_phys = false, bound = false;
  CUdeviceptr uc_va = 0;   // this rank's copy
  CUdeviceptr mc_va = 0;   // stores / reductions here reach every rank's copy
  size_t size = 0;
  int dev = 0;
  int fd = -1;
  ~McRegion();
};

bool multicast_supported(int dev);
// collective over the world's ranks (NCCL barriers inside); `token` is rank 0's
// rendezvous token and `seq` numbers the world's regions (identical everywhere)
McRegion* mcast_create(esp_world_s* w, size_t bytes, uint64_t token, uint32_t seq, cudaStream_t st);

}  // namespace esp
