// NVLink SHARP (NVLS) multicast regions for the fused Allgather (SURVEY.md 8f
// NEXT-1): one multimem store of a rank's payload lands in the
// receive buffer of EVERY GPU of the job through the NVSwitch, instead of n-1
// unicast peer copies that all leave through the sender's own NVLinks.
//
// A region is one multicast object (cuMulticastCreate on rank 0) with one
// physical allocation per rank bound to it, mapped twice on every rank: the
// unicast view (the rank's own copy, read by h2) and the multicast view
// (stores and reductions on it reach every copy).  Rank 0 exports the object
// as a POSIX file descriptor and hands it to the other ranks over an abstract
// unix-domain socket (SCM_RIGHTS); NCCL carries the rendezvous token and the
// barriers.  The CUDA driver API is reached through cudaGetDriverEntryPoint,
// so libesp.so has no link-time dependency on libcuda.
#include <cuda.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <chrono>
#include <cstddef>
#include <thread>

#include "esp_internal.h"
#include "mcast.h"

namespace esp {

namespace {

struct Drv {
  CUresult (*multicastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*multicastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*multicastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long);
  CUresult (*multicastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*multicastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*memRelease)(CUmemGenericAllocationHandle);
  CUresult (*memAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*memAddressFree)(CUdeviceptr, size_t);
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*memUnmap)(CUdeviceptr, size_t);
  CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*memExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long);
  CUresult (*memImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*deviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
  CUresult (*deviceGet)(CUdevice*, int);
  bool ok = false;
};

const Drv& drv() {
  static const Drv d = [] {
    Drv x{};
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q{};
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    x.ok = get("cuMulticastCreate", (void**)&x.multicastCreate) &&
           get("cuMulticastAddDevice", (void**)&x.multicastAddDevice) &&
           get("cuMulticastBindMem", (void**)&x.multicastBindMem) &&
           get("cuMulticastUnbind", (void**)&x.multicastUnbind) &&
           get("cuMulticastGetGranularity", (void**)&x.multicastGetGranularity) &&
           get("cuMemCreate", (void**)&x.memCreate) && get("cuMemRelease", (void**)&x.memRelease) &&
           get("cuMemAddressReserve", (void**)&x.memAddressReserve) &&
           get("cuMemAddressFree", (void**)&x.memAddressFree) && get("cuMemMap", (void**)&x.memMap) &&
           get("cuMemUnmap", (void**)&x.memUnmap) && get("cuMemSetAccess", (void**)&x.memSetAccess) &&
           get("cuMemExportToShareableHandle", (void**)&x.memExportToShareableHandle) &&
           get("cuMemImportFromShareableHandle", (void**)&x.memImportFromShareableHandle) &&
           get("cuDeviceGetAttribute", (void**)&x.deviceGetAttribute) && get("cuDeviceGet", (void**)&x.deviceGet);
    cudaGetLastError();
    return x;
  }();
  return d;
}

#define ESP_CU(x)                                                                    \
  do {                                                                               \
    CUresult r_ = (x);                                                               \
    if (r_ != CUDA_SUCCESS) {                                                        \
      ::esp::set_error(std::string(#x) + ": CUDA driver error " + std::to_string(r_)); \
      throw ::esp::Fail{ESP_ERR_CUDA};                                               \
    }                                                                                \
  } while (0)

// every rank of the world reaches this point (and its stream is drained)
void barrier(esp_world_s* w, cudaStream_t st) {
  int* d = nullptr;
  ESP_CUDA(cudaMallocAsync(&d, sizeof(int), st));
  ESP_CUDA(cudaMemsetAsync(d, 0, sizeof(int), st));
  ESP_NCCL(ncclAllReduce(d, d, 1, ncclInt32, ncclSum, w->comm, st));
  ESP_CUDA(cudaFreeAsync(d, st));
  ESP_CUDA(cudaStreamSynchronize(st));
}

std::string sock_name(uint64_t token, uint32_t seq) {
  char buf[64];
  snprintf(buf, sizeof(buf), "esp-mcast-%016llx-%u", (unsigned long long)token, seq);
  return buf;
}

sockaddr_un sock_addr(const std::string& name, socklen_t* len) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  a.sun_path[0] = '\0';   // abstract namespace: nothing on the file system
  memcpy(a.sun_path + 1, name.data(), name.size());
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + name.size());
  return a;
}

void send_fd(int conn, int fd) {
  char byte = 'F';
  iovec io{&byte, 1};
  alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  memcpy(CMSG_DATA(c), &fd, sizeof(int));
  ESP_REQUIRE(sendmsg(conn, &m, 0) == 1, ESP_ERR_STATE, "multicast: sendmsg of the handle failed");
}

int recv_fd(const std::string& name) {
  socklen_t len = 0;
  const sockaddr_un a = sock_addr(name, &len);
  int s = -1;
  for (int attempt = 0; attempt < 200; ++attempt) {   // the listener exists (barrier), retry transient errors
    s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s >= 0 && connect(s, reinterpret_cast<const sockaddr*>(&a), len) == 0) break;
    if (s >= 0) close(s);
    s = -1;
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
  ESP_REQUIRE(s >= 0, ESP_ERR_STATE, "multicast: cannot reach rank 0's handle socket");
  char byte = 0;
  iovec io{&byte, 1};
  alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  const ssize_t r = recvmsg(s, &m, 0);
  close(s);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  ESP_REQUIRE(r == 1 && c && c->cmsg_type == SCM_RIGHTS, ESP_ERR_STATE, "multicast: no handle received");
  int fd = -1;
  memcpy(&fd, CMSG_DATA(c), sizeof(int));
  return fd;
}

}  // namespace

bool multicast_supported(int dev) {
  const Drv& d = drv();
  if (!d.ok) return false;
  CUdevice cd;
  if (d.deviceGet(&cd, dev) != CUDA_SUCCESS) return false;
  int v = 0;
  return d.deviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) == CUDA_SUCCESS && v != 0;
}

// Collective over the world: every rank calls it with the same bytes.
McRegion* mcast_create(esp_world_s* w, size_t bytes, uint64_t token, uint32_t seq, cudaStream_t st) {
  const Drv& d = drv();
  ESP_REQUIRE(d.ok, ESP_ERR_UNSUPPORTED, "multicast: CUDA driver entry points unavailable");
  const int n = w->nranks;
  auto r = std::make_unique<McRegion>();
  CUdevice dev;
  ESP_CU(d.deviceGet(&dev, w->dev));
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)n;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  size_t gran = 0;
  ESP_CU(d.multicastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  r->size = (bytes + gran - 1) / gran * gran;
  mp.size = r->size;
  // rank 0 creates the object and serves its handle; the others fetch it
  const std::string name = sock_name(token, seq);
  int listener = -1;
  if (w->rank == 0) {
    ESP_CU(d.multicastCreate(&r->mc, &mp));
    r->have_mc = true;
    int fd = -1;
    ESP_CU(d.memExportToShareableHandle(&fd, r->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    r->fd = fd;
    socklen_t len = 0;
    const sockaddr_un a = sock_addr(name, &len);
    listener = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    ESP_REQUIRE(listener >= 0 && bind(listener, reinterpret_cast<const sockaddr*>(&a), len) == 0 &&
                    listen(listener, n) == 0,
                ESP_ERR_STATE, "multicast: cannot open the handle socket");
  }
  barrier(w, st);   // the socket is listening
  if (w->rank == 0) {
    for (int q = 1; q < n; ++q) {
      const int conn = accept(listener, nullptr, nullptr);
      ESP_REQUIRE(conn >= 0, ESP_ERR_STATE, "multicast: accept failed");
      send_fd(conn, r->fd);
      close(conn);
    }
    close(listener);
  } else {
    r->fd = recv_fd(name);
    ESP_CU(d.memImportFromShareableHandle(&r->mc, reinterpret_cast<void*>((uintptr_t)r->fd),
                                         CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    r->have_mc = true;
  }
  ESP_CU(d.multicastAddDevice(r->mc, dev));
  barrier(w, st);   // every device is in the team before memory is bound
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = w->dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;   // as the multicast object's
  ESP_CU(d.memCreate(&r->phys, r->size, &ap, 0));
  r->have_phys = true;
  ESP_CU(d.multicastBindMem(r->mc, 0, r->phys, 0, r->size, 0));
  r->bound = true;
  CUmemAccessDesc ad{};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = w->dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  ESP_CU(d.memAddressReserve(&r->uc_va, r->size, gran, 0, 0));
  ESP_CU(d.memMap(r->uc_va, r->size, 0, r->phys, 0));
  ESP_CU(d.memSetAccess(r->uc_va, r->size, &ad, 1));
  ESP_CU(d.memAddressReserve(&r->mc_va, r->size, gran, 0, 0));
  ESP_CU(d.memMap(r->mc_va, r->size, 0, r->mc, 0));
  ESP_CU(d.memSetAccess(r->mc_va, r->size, &ad, 1));
  r->dev = w->dev;
  ESP_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(r->uc_va), 0, r->size, st));
  barrier(w, st);   // bound and zeroed everywhere before any multicast store
  return r.release();
}

McRegion::~McRegion() {
  const Drv& d = drv();
  if (!d.ok) return;
  cudaDeviceSynchronize();
  if (mc_va) {
    d.memUnmap(mc_va, size);
    d.memAddressFree(mc_va, size);
  }
  if (uc_va) {
    d.memUnmap(uc_va, size);
    d.memAddressFree(uc_va, size);
  }
  if (bound) {
    CUdevice cd;
    if (d.deviceGet(&cd, dev) == CUDA_SUCCESS) d.multicastUnbind(mc, cd, 0, size);
  }
  if (have_phys) d.memRelease(phys);
  if (have_mc) d.memRelease(mc);
  if (fd >= 0) close(fd);
}

}  // namespace esp
