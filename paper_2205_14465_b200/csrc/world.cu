// Worlds and the collective layer (NCCL inside a
// machine, a CCL per data format, several CUDA streams).  A world is either an
// NCCL communicator (one process per GPU, NVLink 5 / NVSwitch) or a "sim" world
// of n virtual ranks on one GPU whose collectives are device-to-device copies.
#include <cstdlib>
#include <atomic>
#include <cmath>

#include "esp_internal.h"
#include "esp_kernels.h"

namespace esp {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

uint64_t host_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---- sizes ---------------------------------------------------------------------
uint32_t k_of(uint64_t numel, double ratio) {
  if (numel == 0) return 0;
  double c = std::ceil(ratio * (double)numel);   // R1: max(1, ceil(rho N)), <= N
  uint64_t k = c < 1.0 ? 1 : (uint64_t)c;
  return (uint32_t)(k > numel ? numel : k);
}

int nparts_of(int routine, int n) { return routine == ESP_ALLTOALL_ALLGATHER ? n : 1; }

uint32_t partition_len(uint64_t numel, int nparts) {
  if (nparts == 1) return (uint32_t)numel;
  uint64_t L = (numel + nparts - 1) / nparts;
  return (uint32_t)round_up(L, 32);   // R10
}

bool is_sparse(int kind) { return kind == ESP_RANDOMK || kind == ESP_DGC || kind == ESP_TOPK; }
bool is_quant(int kind) { return kind == ESP_EFSIGNSGD || kind == ESP_ONEBIT; }
int process_of(const esp_compressor_cfg_t& cfg) {
  if (cfg.process == 1 || cfg.process == 2) return cfg.process;
  return is_sparse(cfg.kind) ? 1 : 2;   // the cost table's choice
}
bool mid_scheme(const esp_compressor_cfg_t& cfg, int routine) {
  return cfg.kind != ESP_NONE && process_of(cfg) == 2 &&
         (routine == ESP_ALLTOALL_ALLGATHER || routine == ESP_GATHER_BROADCAST);
}

bool pair_legal(const esp_compressor_cfg_t& cfg, int routine) {
  // routines table; "cannot use Allreduce" P:1073; allreducible P:38/P:56
  if (cfg.kind == ESP_NONE)
    return routine == ESP_ALLREDUCE || routine == ESP_REDUCESCATTER_ALLGATHER ||
           routine == ESP_REDUCE_BROADCAST;
  if (routine == ESP_ALLGATHER || routine == ESP_ALLTOALL_ALLGATHER || routine == ESP_GATHER_BROADCAST)
    return true;
  return cfg.kind == ESP_RANDOMK && cfg.randomk_shared_indices && routine == ESP_ALLREDUCE;
}

size_t chunk_bytes_of(const esp_compressor_cfg_t& cfg, uint64_t numel, int nparts, uint32_t* kpad_out) {
  const uint64_t L = partition_len(numel, nparts);
  uint64_t maxlen = 0, maxk = 0;
  for (int p = 0; p < nparts; ++p) {
    uint64_t lo = std::min<uint64_t>(numel, (uint64_t)p * L), hi = std::min<uint64_t>(numel, lo + L);
    if (nparts == 1) { lo = 0; hi = numel; }
    maxlen = std::max(maxlen, hi - lo);
    maxk = std::max<uint64_t>(maxk, k_of(hi - lo, cfg.ratio));
  }
  uint32_t kpad = 0;
  size_t bytes = 0;
  switch (cfg.kind) {
    case ESP_DGC: case ESP_TOPK:
      kpad = (uint32_t)round_up(maxk, 4); bytes = 8ull * kpad; break;
    case ESP_RANDOMK:
      kpad = (uint32_t)round_up(maxk, 4); bytes = 4ull * kpad; break;
    case ESP_EFSIGNSGD: case ESP_ONEBIT:
      kpad = (uint32_t)round_up((maxlen + 31) / 32, 4); bytes = 16 + 4ull * kpad; break;
    default:
      kpad = 0; bytes = 4ull * numel; break;
  }
  if (kpad_out) *kpad_out = kpad;
  return bytes;
}

void Arena::alloc() {
  size = round_up(used, 256);
  if (size) ESP_CUDA(cudaMalloc(&base, size));
}
Arena::~Arena() {
  if (base) cudaFree(base);
}

// ---- collectives (the *_f32 reductions are counted by the caller with logical sizes) -----------------------------------------------------------------
void count_coll(esp_world_s* w, int lr, int op, uint64_t sent, uint64_t recv) {
  esp_counters_t& c = w->counters[lr];
  c.calls[op] += 1;
  c.sent[op] += sent;
  c.recv[op] += recv;
}
static int grank(esp_world_s* w, int lr) { return w->sim ? lr : w->rank; }

static void d2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes && dst != src) ESP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
}
// one real rank: the plan aliases receive and send buffers, nothing moves
static bool solo(esp_world_s* w) { return !w->sim && w->nranks == 1; }

void coll_allgather(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t bytes, cudaStream_t st) {
  const int n = w->nranks;
  for (int lr = 0; lr < w->nlocal; ++lr) count_coll(w, lr, ESP_OP_ALLGATHER, (n - 1) * bytes, (n - 1) * bytes);
  if (solo(w)) {
    d2d(recv.at(0), send.at(0), bytes, st);
    return;
  }
  if (w->sim) {
    for (int q = 0; q < n; ++q)
      for (int r = 0; r < n; ++r) d2d(recv.at(q) + r * bytes, send.at(r), bytes, st);
  } else {
    ESP_NCCL(ncclAllGather(send.at(0), recv.at(0), bytes, ncclUint8, w->comm, st));
  }
}

void coll_alltoall(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t chunk, cudaStream_t st) {
  const int n = w->nranks;
  for (int lr = 0; lr < w->nlocal; ++lr) count_coll(w, lr, ESP_OP_ALLTOALL, (n - 1) * chunk, (n - 1) * chunk);
  if (solo(w)) {
    d2d(recv.at(0), send.at(0), chunk, st);
    return;
  }
  if (w->sim) {
    for (int q = 0; q < n; ++q)
      for (int r = 0; r < n; ++r) d2d(recv.at(q) + r * chunk, send.at(r) + q * chunk, chunk, st);
  } else {
    ESP_NCCL(ncclAlltoAll(send.at(0), recv.at(0), chunk, ncclUint8, w->comm, st));
  }
}

void coll_gather(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t bytes, cudaStream_t st) {
  const int n = w->nranks;
  for (int lr = 0; lr < w->nlocal; ++lr) {
    if (grank(w, lr) == 0) count_coll(w, lr, ESP_OP_GATHER, 0, (n - 1) * bytes);
    else count_coll(w, lr, ESP_OP_GATHER, bytes, 0);
  }
  if (solo(w)) {
    d2d(recv.at(0), send.at(0), bytes, st);
    return;
  }
  if (w->sim) {
    for (int r = 0; r < n; ++r) d2d(recv.at(0) + r * bytes, send.at(r), bytes, st);
  } else {
    ESP_NCCL(ncclGather(send.at(0), recv.at(0), bytes, ncclUint8, 0, w->comm, st));
  }
}

void coll_broadcast(esp_world_s* w, LocalBufs buf, size_t bytes, cudaStream_t st) {
  const int n = w->nranks;
  for (int lr = 0; lr < w->nlocal; ++lr) {
    if (grank(w, lr) == 0) count_coll(w, lr, ESP_OP_BROADCAST, n > 1 ? bytes : 0, 0);
    else count_coll(w, lr, ESP_OP_BROADCAST, 0, bytes);
  }
  if (solo(w)) {
    return;
  }
  if (w->sim) {
    for (int q = 1; q < n; ++q) d2d(buf.at(q), buf.at(0), bytes, st);
  } else {
    ESP_NCCL(ncclBroadcast(buf.at(0), buf.at(0), bytes, ncclUint8, 0, w->comm, st));
  }
}

void coll_allreduce_f32(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t count_, cudaStream_t st) {
  if (solo(w)) {
    d2d(recv.at(0), send.at(0), 4 * count_, st);
    return;
  }
  ESP_REQUIRE(!w->sim, ESP_ERR_STATE, "allreduce in a sim world is executed by h2");
  ESP_NCCL(ncclAllReduce(send.at(0), recv.at(0), count_, ncclFloat32, ncclSum, w->comm, st));
}

void coll_reducescatter_f32(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t count_, cudaStream_t st) {
  if (solo(w)) {
    d2d(recv.at(0), send.at(0), 4 * count_, st);
    return;
  }
  ESP_REQUIRE(!w->sim, ESP_ERR_STATE, "reduce-scatter in a sim world is executed by h2");
  ESP_NCCL(ncclReduceScatter(send.at(0), recv.at(0), count_ / w->nranks, ncclFloat32, ncclSum, w->comm, st));
}

void coll_allgather_inplace_f32(esp_world_s* w, LocalBufs buf, size_t count_per_rank, cudaStream_t st) {
  if (solo(w)) {
    return;
  }
  ESP_REQUIRE(!w->sim, ESP_ERR_STATE, "in-place allgather in a sim world is executed by h2");
  float* base = reinterpret_cast<float*>(buf.at(0));
  ESP_NCCL(ncclAllGather(base + (size_t)w->rank * count_per_rank, base, count_per_rank, ncclFloat32,
                         w->comm, st));
}

void coll_reduce_f32(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t count_, cudaStream_t st) {
  if (solo(w)) {
    d2d(recv.at(0), send.at(0), 4 * count_, st);
    return;
  }
  ESP_REQUIRE(!w->sim, ESP_ERR_STATE, "reduce in a sim world is executed by h2");
  ESP_NCCL(ncclReduce(send.at(0), recv.at(0), count_, ncclFloat32, ncclSum, 0, w->comm, st));
}

}  // namespace esp

using namespace esp;

extern "C" {

const char* esp_status_string(esp_status_t s) {
  switch (s) {
    case ESP_OK: return "ESP_OK";
    case ESP_ERR_INVALID_ARG: return "ESP_ERR_INVALID_ARG";
    case ESP_ERR_UNSUPPORTED: return "ESP_ERR_UNSUPPORTED";
    case ESP_ERR_TOO_LARGE: return "ESP_ERR_TOO_LARGE";
    case ESP_ERR_CUDA: return "ESP_ERR_CUDA";
    case ESP_ERR_NCCL: return "ESP_ERR_NCCL";
    case ESP_ERR_OOM: return "ESP_ERR_OOM";
    case ESP_ERR_STATE: return "ESP_ERR_STATE";
  }
  return "ESP_ERR_UNKNOWN";
}

const char* esp_last_error(void) { return g_last_error.c_str(); }
uint64_t esp_launch_count(void) { return g_launches.load(); }
const char* esp_version(void) { return "espresso-b200 0.1 (sm_100a)"; }

esp_status_t esp_get_nccl_unique_id(void* out128) {
  ESP_API_BEGIN
  ESP_REQUIRE(out128, ESP_ERR_INVALID_ARG, "out128 is NULL");
  ncclUniqueId id;
  ESP_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  ESP_API_END
}

static void world_common_init(esp_world_s* w) {
  ESP_CUDA(cudaSetDevice(w->dev));
  int lo = 0, hi = 0;
  ESP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // communication gets the higher priority so collectives are not starved by
  // the next bucket's compression kernels (SURVEY.md 7 hard part 7)
  ESP_CUDA(cudaStreamCreateWithPriority(&w->comm_stream, cudaStreamNonBlocking, hi));
  ESP_CUDA(cudaStreamCreateWithFlags(&w->cap_stream, cudaStreamNonBlocking));
  ESP_CUDA(cudaStreamCreateWithPriority(&w->fin_stream, cudaStreamNonBlocking, hi));
  ESP_CUDA(cudaEventCreateWithFlags(&w->ev_join, cudaEventDisableTiming));
  ESP_CUDA(cudaEventCreateWithFlags(&w->ev_fork, cudaEventDisableTiming));
  w->counters.assign(w->nlocal, esp_counters_t{});
  ESP_CUDA(cudaHostAlloc(&w->wait_err_host, sizeof(unsigned int), cudaHostAllocMapped));
  *w->wait_err_host = 0;
  ESP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&w->wait_err), w->wait_err_host, 0));
}

esp_status_t esp_world_create_nccl(const void* id128, int nranks, int rank, int cuda_dev, esp_world_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(id128 && out, ESP_ERR_INVALID_ARG, "null argument");
  ESP_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks && cuda_dev >= 0, ESP_ERR_INVALID_ARG,
              "bad nranks/rank/device");
  auto w = std::make_unique<esp_world_s>();
  w->sim = false;
  w->nranks = nranks;
  w->rank = rank;
  w->nlocal = 1;
  w->dev = cuda_dev;
  world_common_init(w.get());
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  ESP_NCCL(ncclCommInitRank(&w->comm, nranks, id, rank));
  *out = w.release();
  ESP_API_END
}

esp_status_t esp_world_create_sim(int nranks, int cuda_dev, esp_world_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(out, ESP_ERR_INVALID_ARG, "out is NULL");
  ESP_REQUIRE(nranks >= 1 && nranks <= 64 && cuda_dev >= 0, ESP_ERR_INVALID_ARG, "bad nranks/device");
  auto w = std::make_unique<esp_world_s>();
  w->sim = true;
  w->nranks = nranks;
  w->rank = 0;
  w->nlocal = nranks;
  w->dev = cuda_dev;
  world_common_init(w.get());
  *out = w.release();
  ESP_API_END
}

esp_status_t esp_world_create_loopback(int nranks, int cuda_dev, esp_world_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(out, ESP_ERR_INVALID_ARG, "out is NULL");
  ESP_REQUIRE(nranks >= 2 && nranks <= 64 && cuda_dev >= 0, ESP_ERR_INVALID_ARG, "bad nranks/device");
  std::vector<std::unique_ptr<esp_world_s>> ws;
  for (int r = 0; r < nranks; ++r) {
    auto w = std::make_unique<esp_world_s>();
    w->loopback = true;
    w->nranks = nranks;
    w->rank = r;
    w->nlocal = 1;
    w->dev = cuda_dev;
    w->wait_timeout_ns = 5ull * 1000000000ull;   // every wait is satisfied at launch: 5 s means a bug
    world_common_init(w.get());
    ws.push_back(std::move(w));
  }
  for (int r = 0; r < nranks; ++r) out[r] = ws[r].release();
  ESP_API_END
}

// a world object with its streams and events (no communicator yet)
static std::unique_ptr<esp_world_s> make_world(int nranks, int rank, int dev, bool loopback) {
  auto w = std::make_unique<esp_world_s>();
  w->loopback = loopback;
  w->nranks = nranks;
  w->rank = rank;
  w->nlocal = 1;
  w->dev = dev;
  if (loopback) w->wait_timeout_ns = 5ull * 1000000000ull;
  world_common_init(w.get());
  return w;
}

esp_status_t esp_world_create_hier(esp_world_t parent, int group, esp_world_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(parent && out, ESP_ERR_INVALID_ARG, "null argument");
  ESP_REQUIRE(parent->comm && !parent->sim && !parent->loopback && parent->hier_g == 0, ESP_ERR_STATE,
              "a hierarchical world splits a flat NCCL world");
  const int n = parent->nranks;
  ESP_REQUIRE(group >= 1 && n % group == 0, ESP_ERR_INVALID_ARG, "group must divide the number of ranks");
  ESP_CUDA(cudaSetDevice(parent->dev));
  const int a = parent->rank / group, i = parent->rank % group, m = n / group;
  auto w = make_world(n, parent->rank, parent->dev, false);
  w->hier_g = group;
  auto intra = make_world(group, i, parent->dev, false);
  auto inter = make_world(m, a, parent->dev, false);
  // machine = color a (key i), inter-machine group = color i (key a); both
  // splits are collective over the parent communicator, in this order
  ESP_NCCL(ncclCommSplit(parent->comm, a, i, &intra->comm, nullptr));
  ESP_NCCL(ncclCommSplit(parent->comm, i, a, &inter->comm, nullptr));
  w->intra = intra.release();
  w->inter = inter.release();
  *out = w.release();
  ESP_API_END
}

esp_status_t esp_world_create_loopback_hier(int nranks, int group, int cuda_dev, esp_world_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(out, ESP_ERR_INVALID_ARG, "out is NULL");
  ESP_REQUIRE(nranks >= 2 && nranks <= 64 && group >= 1 && nranks % group == 0 && cuda_dev >= 0,
              ESP_ERR_INVALID_ARG, "bad nranks/group/device");
  const int m = nranks / group;
  std::vector<std::unique_ptr<esp_world_s>> ws;
  for (int r = 0; r < nranks; ++r) {
    auto w = make_world(nranks, r, cuda_dev, true);
    w->hier_g = group;
    // the machine's phases address each other's arenas directly; the
    // inter-machine group of local index i is a loopback group of m ranks
    // (a single rank: a solo world, its collectives are identities)
    w->intra = make_world(group, r % group, cuda_dev, true).release();
    w->inter = make_world(m, r / group, cuda_dev, m > 1).release();
    ws.push_back(std::move(w));
  }
  for (int r = 0; r < nranks; ++r) out[r] = ws[r].release();
  ESP_API_END
}

esp_status_t esp_world_destroy(esp_world_t w) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  ESP_REQUIRE(w->ctxs.empty(), ESP_ERR_STATE, "destroy every ctx of the world first");
  cudaSetDevice(w->dev);
  cudaStreamSynchronize(w->comm_stream);
  clear_hier_plans(w);
  if (w->intra) esp_world_destroy(w->intra);
  if (w->inter) esp_world_destroy(w->inter);
  clear_plans(w);
  if (w->comm) ncclCommDestroy(w->comm);
  for (auto e : w->tev) cudaEventDestroy(e);
  for (auto e : w->probe_pool) cudaEventDestroy(e);
  cudaEventDestroy(w->ev_join);
  cudaEventDestroy(w->ev_fork);
  if (w->wait_err_host) cudaFreeHost(w->wait_err_host);
  cudaStreamDestroy(w->comm_stream);
  cudaStreamDestroy(w->cap_stream);
  cudaStreamDestroy(w->fin_stream);
  delete w;
  ESP_API_END
}

esp_status_t esp_world_check(esp_world_t w) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  cudaError_t e = cudaGetLastError();
  ESP_REQUIRE(e == cudaSuccess, ESP_ERR_CUDA, std::string("async CUDA error: ") + cudaGetErrorString(e));
  ESP_REQUIRE(!*const_cast<volatile unsigned int*>(w->wait_err_host), ESP_ERR_NCCL,
              "a peer's payload did not arrive within the wait timeout (esp_world_set_timeout)");
  if (w->comm) {
    ncclResult_t r = ncclSuccess;
    ESP_NCCL(ncclCommGetAsyncError(w->comm, &r));
    ESP_REQUIRE(r == ncclSuccess || r == ncclInProgress, ESP_ERR_NCCL,
                std::string("async NCCL error: ") + ncclGetErrorString(r));
  }
  ESP_API_END
}

esp_status_t esp_world_info(esp_world_t w, int* nranks, int* rank, int* nlocal) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  if (nranks) *nranks = w->nranks;
  if (rank) *rank = w->rank;
  if (nlocal) *nlocal = w->nlocal;
  ESP_API_END
}

esp_status_t esp_world_counters(esp_world_t w, esp_counters_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && out, ESP_ERR_INVALID_ARG, "null argument");
  *out = w->counters[0];
  ESP_API_END
}

esp_status_t esp_world_counters_local(esp_world_t w, int lr, esp_counters_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && out && lr >= 0 && lr < w->nlocal, ESP_ERR_INVALID_ARG, "bad argument");
  *out = w->counters[lr];
  ESP_API_END
}

esp_status_t esp_world_reset_counters(esp_world_t w) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  w->counters.assign(w->nlocal, esp_counters_t{});
  ESP_API_END
}

esp_status_t esp_world_set_timing(esp_world_t w, int enable) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  w->timing = enable != 0;
  ESP_API_END
}

esp_status_t esp_world_set_bucket_elems(esp_world_t w, uint64_t elems) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  w->bucket_elems = elems;
  clear_plans(w);
  if (w->inter) esp_world_set_bucket_elems(w->inter, elems);
  ESP_API_END
}

esp_status_t esp_world_set_timeout(esp_world_t w, double seconds) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && seconds > 0 && seconds < 1e9, ESP_ERR_INVALID_ARG, "bad argument");
  w->wait_timeout_ns = (unsigned long long)(seconds * 1e9);
  ESP_API_END
}

esp_status_t esp_world_set_plan_cache(esp_world_t w, int max_plans) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && max_plans >= 1, ESP_ERR_INVALID_ARG, "bad argument");
  w->plan_cap = (size_t)max_plans;
  trim_plans(w);
  ESP_API_END
}

esp_status_t esp_world_set_multicast(esp_world_t w, int mode) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && mode >= -1 && mode <= 1, ESP_ERR_INVALID_ARG, "mode must be -1, 0 or 1");
  cudaSetDevice(w->dev);
  clear_plans(w);
  w->mc_mode = mode;
  ESP_API_END
}

esp_status_t esp_world_drop_plans(esp_world_t w) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  cudaSetDevice(w->dev);
  clear_plans(w);
  ESP_API_END
}

esp_status_t esp_world_set_probe(esp_world_t w, int enable) {
  ESP_API_BEGIN
  ESP_REQUIRE(w, ESP_ERR_INVALID_ARG, "world is NULL");
  w->probe = enable != 0;
  w->probe_used = 0;
  if (w->inter) esp_world_set_probe(w->inter, enable);   // hierarchical: the h1 kernels run in the inter world
  ESP_API_END
}

esp_status_t esp_probe_read(esp_world_t w, double* ms, uint64_t* launches, uint64_t* bytes) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && ms && launches && bytes, ESP_ERR_INVALID_ARG, "null argument");
  if (w->inter) return esp_probe_read(w->inter, ms, launches, bytes);
  double t = 0;
  uint64_t b = 0;
  for (size_t i = 0; i < w->probe_used; ++i) {
    ESP_CUDA(cudaEventSynchronize(w->probe_pool[2 * i + 1]));
    float x = 0;
    ESP_CUDA(cudaEventElapsedTime(&x, w->probe_pool[2 * i], w->probe_pool[2 * i + 1]));
    t += x;
    b += w->probe_bytes[i];
  }
  *ms = t;
  *launches = w->probe_used;
  *bytes = b;
  w->probe_used = 0;
  ESP_API_END
}

esp_status_t esp_compressed_bytes(const esp_compressor_cfg_t* cfg, size_t numel, int nparts, size_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(cfg && out && nparts >= 1, ESP_ERR_INVALID_ARG, "bad argument");
  ESP_REQUIRE(cfg->kind >= ESP_NONE && cfg->kind <= ESP_ONEBIT, ESP_ERR_INVALID_ARG, "bad kind");
  ESP_REQUIRE(numel < (1ull << 31), ESP_ERR_TOO_LARGE, "numel >= 2^31");
  *out = chunk_bytes_of(*cfg, numel, nparts, nullptr) * (size_t)nparts;
  ESP_API_END
}

esp_status_t esp_wire_bytes(int routine, int tensor_type, double M, int n, double* sent, double* recv) {
  ESP_API_BEGIN
  ESP_REQUIRE(sent && recv && n >= 1 && M >= 0 && routine >= ESP_ALLREDUCE && routine <= ESP_REDUCE_BROADCAST &&
                  tensor_type >= ESP_TT_ALLREDUCIBLE && tensor_type <= ESP_TT_QUANTIZED,
              ESP_ERR_INVALID_ARG, "bad argument");
  const bool allred = tensor_type == ESP_TT_ALLREDUCIBLE;
  const bool uncompressed_routine = routine == ESP_ALLREDUCE || routine == ESP_REDUCESCATTER_ALLGATHER ||
                                    routine == ESP_REDUCE_BROADCAST;
  ESP_REQUIRE(allred == uncompressed_routine, ESP_ERR_UNSUPPORTED,
              "allreducible data takes Allreduce, Reduce-scatter/Allgather or Reduce/Broadcast; compressed "
              "payloads the other routines (P:1064-1065, P:1073)");
  // cost table of flat communication, P:38-43 (communication volume = time * B);
  // the uncompressed pairs per S:126
  double v = 0;
  if (n > 1) {
    const bool q = tensor_type == ESP_TT_QUANTIZED;
    switch (routine) {
      case ESP_ALLREDUCE: v = 2.0 * (n - 1) * M / n; break;
      case ESP_REDUCESCATTER_ALLGATHER: v = (n - 1) * M / n + (n - 1) * (M / n); break;
      case ESP_REDUCE_BROADCAST: v = (n - 1) * M + M; break;
      case ESP_ALLGATHER: v = (n - 1) * M; break;
      case ESP_ALLTOALL_ALLGATHER: v = q ? 2.0 * (n - 1) * M / n : ((double)n * n - 1) * M / n; break;   // R13
      default: v = q ? (double)n * M : (2.0 * n - 1) * M; break;                                   // G/B
    }
  }
  *sent = v;
  *recv = v;
  ESP_API_END
}

esp_status_t esp_curve_eval(const esp_curve_t* c, double bytes, double* out_seconds) {
  ESP_API_BEGIN
  ESP_REQUIRE(c && out_seconds && c->n >= 1 && c->bytes && c->seconds && bytes > 0, ESP_ERR_INVALID_ARG,
              "bad curve");
  for (int i = 0; i < c->n; ++i) {
    ESP_REQUIRE(c->bytes[i] > 0 && c->seconds[i] > 0, ESP_ERR_INVALID_ARG, "curve samples must be positive");
    if (i) ESP_REQUIRE(c->bytes[i] > c->bytes[i - 1], ESP_ERR_INVALID_ARG, "curve sizes must increase");
  }
  // log-log piecewise-linear; clamp below the first sample (launch floor),
  // extend the last segment above the last sample
  if (c->n == 1 || bytes <= c->bytes[0]) {   // one sample: a constant
    *out_seconds = c->seconds[0];
    return ESP_OK;
  }
  int i = 1;
  while (i < c->n - 1 && bytes > c->bytes[i]) ++i;
  const double x0 = std::log(c->bytes[i - 1]), x1 = std::log(c->bytes[i]);
  const double y0 = std::log(c->seconds[i - 1]), y1 = std::log(c->seconds[i]);
  const double x = std::log(bytes);
  *out_seconds = std::exp(y0 + (y1 - y0) * (x - x0) / (x1 - x0));
  ESP_API_END
}

esp_status_t esp_option_time(const esp_option_t* o, size_t numel, int n, double B, double* out_seconds) {
  ESP_API_BEGIN
  ESP_REQUIRE(o && out_seconds && n >= 1 && B > 0 && numel >= 1, ESP_ERR_INVALID_ARG, "bad argument");
  ESP_REQUIRE(numel < (1ull << 31), ESP_ERR_TOO_LARGE, "numel >= 2^31");
  ESP_REQUIRE(pair_legal(o->cfg, o->routine), ESP_ERR_UNSUPPORTED, "illegal (compressor, routine) pair");
  const double in_bytes = 4.0 * (double)numel;
  if (o->cfg.kind == ESP_NONE) {
    // uncompressed: communication only.  Allreduce and Reduce-scatter +
    // Allgather move 2(n-1)M/n; Reduce (n-1)M then Broadcast of
    // the M-byte result M: nM
    double v = 0.0;
    if (n > 1) v = o->routine == ESP_REDUCE_BROADCAST ? (double)n * in_bytes : 2.0 * (n - 1) * in_bytes / n;
    *out_seconds = v / B;
    return ESP_OK;
  }
  const int P = nparts_of(o->routine, n);
  const double M = (double)chunk_bytes_of(o->cfg, numel, P, nullptr) * P;
  const bool p2 = mid_scheme(o->cfg, o->routine);
  int row = 0;
  switch (o->routine) {
    case ESP_ALLREDUCE: row = 0; break;
    case ESP_ALLGATHER: row = 1; break;
    case ESP_ALLTOALL_ALLGATHER: row = p2 ? 3 : 2; break;
    default: row = p2 ? 5 : 4; break;   // Gather/Broadcast
  }
  const int tt = row == 0 ? ESP_TT_ALLREDUCIBLE : (p2 ? ESP_TT_QUANTIZED : ESP_TT_SPARSE);
  double comm = 0;
  esp_status_t s = esp_model_time(o->routine, tt, M, n, B, &comm);
  if (s != ESP_OK) return s;
  auto ev = [&](const esp_curve_t& c, double b) {
    double t = 0;
    const esp_status_t e = esp_curve_eval(&c, b, &t);
    ESP_REQUIRE(e == ESP_OK, e, "bad cost curve");
    return t;
  };
  const double part = in_bytes / n;
  double comp = 0;
  switch (row) {   // compression column of P:38-43 (R12: Gather/Broadcast quantized decodes h2(M))
    case 0: comp = ev(o->h1, in_bytes) + ev(o->h2, in_bytes); break;
    case 1: comp = ev(o->h1, in_bytes) + n * ev(o->h2, in_bytes); break;
    case 2: comp = ev(o->h1, in_bytes) + (double)n * n * ev(o->h2, part); break;
    case 3: comp = ev(o->h1, in_bytes) + ev(o->h1, part) + 2.0 * n * ev(o->h2, part); break;
    case 4: comp = ev(o->h1, in_bytes) + n * ev(o->h2, in_bytes); break;
    default: comp = 2.0 * ev(o->h1, in_bytes) + (n + 1.0) * ev(o->h2, in_bytes); break;
  }
  *out_seconds = comm + comp;
  ESP_API_END
}

esp_status_t esp_select_option(const esp_option_t* opts, int nopt, size_t numel, int n, double B, int* best,
                               double* out_seconds) {
  ESP_API_BEGIN
  ESP_REQUIRE(opts && nopt >= 1 && best && out_seconds, ESP_ERR_INVALID_ARG, "bad argument");
  int bi = -1;
  double bt = 0;
  for (int i = 0; i < nopt; ++i) {
    double t = 0;
    const esp_status_t s = esp_option_time(opts + i, numel, n, B, &t);
    if (s != ESP_OK) return s;
    if (bi < 0 || t < bt) {
      bi = i;
      bt = t;
    }
  }
  *best = bi;
  *out_seconds = bt;
  ESP_API_END
}

esp_status_t esp_model_time(int routine, int tensor_type, double M, int n, double B, double* out_seconds) {
  ESP_API_BEGIN
  ESP_REQUIRE(out_seconds && B > 0, ESP_ERR_INVALID_ARG, "bad argument");
  double sent = 0, recv = 0;
  esp_status_t s = esp_wire_bytes(routine, tensor_type, M, n, &sent, &recv);
  if (s != ESP_OK) return s;
  *out_seconds = recv / B;
  ESP_API_END
}

}  // extern "C"
