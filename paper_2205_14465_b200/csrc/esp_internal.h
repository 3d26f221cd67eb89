// Host-side runtime of libesp: worlds, per-tensor contexts, cached execution
// plans (bucketing + device work tables), and the collective layer.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../../include/esp.h"
#include "esp_tables.h"

namespace esp {

// ---- error plumbing (thread-local last error; never throw across the ABI) ----
void set_error(const std::string& msg);
struct Fail {
  esp_status_t st;
};
#define ESP_CUDA(x)                                                             \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      ::esp::set_error(std::string(#x) + ": " + cudaGetErrorString(e_));        \
      throw ::esp::Fail{e_ == cudaErrorMemoryAllocation ? ESP_ERR_OOM : ESP_ERR_CUDA}; \
    }                                                                           \
  } while (0)
#define ESP_NCCL(x)                                                             \
  do {                                                                          \
    ncclResult_t r_ = (x);                                                      \
    if (r_ != ncclSuccess) {                                                    \
      ::esp::set_error(std::string(#x) + ": " + ncclGetErrorString(r_));        \
      throw ::esp::Fail{ESP_ERR_NCCL};                                          \
    }                                                                           \
  } while (0)
#define ESP_REQUIRE(cond, code, msg)                                            \
  do {                                                                          \
    if (!(cond)) {                                                              \
      ::esp::set_error(msg);                                                    \
      throw ::esp::Fail{code};                                                  \
    }                                                                           \
  } while (0)

uint64_t host_splitmix64(uint64_t z);
void count_coll(esp_world_s* w, int lr, int op, uint64_t sent, uint64_t recv);
inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline uint32_t div_up(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }

// ---- sizes (reading R1, R10; independent of the oracle) ----
uint32_t k_of(uint64_t numel, double ratio);
uint32_t partition_len(uint64_t numel, int nparts);   // L (multiple of 32) or numel
int nparts_of(int routine, int n);
bool is_sparse(int kind);
bool is_quant(int kind);
// process 1 / 2 of the divisible routines (R19; 0 -> sparse 1, quantized 2)
int process_of(const esp_compressor_cfg_t& cfg);
// a divisible routine in process 2: decompress-aggregate-recompress mid-scheme (a7)
bool mid_scheme(const esp_compressor_cfg_t& cfg, int routine);
bool pair_legal(const esp_compressor_cfg_t& cfg, int routine);
size_t chunk_bytes_of(const esp_compressor_cfg_t& cfg, uint64_t numel, int nparts,
                      uint32_t* kpad_out);

// ---- device memory arena (one cudaMalloc, 256 B aligned sub-allocations) ----
struct Arena {
  unsigned char* base = nullptr;
  size_t size = 0, used = 0;
  size_t reserve(size_t bytes) {   // returns offset
    size_t off = round_up(used, 256);
    used = off + bytes;
    return off;
  }
  void alloc();
  ~Arena();
};

struct Plan;
struct HierPlan;

}  // namespace esp

struct esp_world_s {
  bool sim = false;
  bool loopback = false;                   // one of n worlds of one process acting as ranks (tests)
  int nranks = 1, rank = 0, nlocal = 1, dev = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaStream_t cap_stream = nullptr;       // CUDA-graph capture of a plan's call (non-blocking)
  cudaStream_t fin_stream = nullptr;       // DGC finalize chains of a multi-bucket call (a9)
  cudaEvent_t ev_join = nullptr, ev_fork = nullptr;
  std::vector<esp_counters_t> counters;   // per local rank
  bool timing = false;
  esp_timing_t last{};
  std::vector<cudaEvent_t> tev;            // timing events of the last call
  uint64_t bucket_elems = 0;
  // dominant-kernel probe (bench roofline): event pairs recorded around the
  // streaming h1 kernel of every bucket, with the algorithmic bytes it moves
  bool probe = false;
  std::vector<cudaEvent_t> probe_pool;
  size_t probe_used = 0;
  std::vector<uint64_t> probe_bytes;
  std::vector<esp::Plan*> plans;           // owned; freed by esp::clear_plans (LRU order, most recent last)
  int mc_mode = -1;                        // NVLS multicast for fused Allgather: -1 auto (n >= 3), 0 off, 1 on
  uint32_t mc_seq = 0;                     // multicast regions created (rendezvous names)
  size_t plan_cap = 64;                    // cached plans kept per world (least recently used evicted)
  // fused collectives: a wait kernel that saw no arrival within wait_timeout_ns
  // sets the mapped word *wait_err_host (device alias wait_err)
  unsigned int* wait_err_host = nullptr;
  unsigned int* wait_err = nullptr;
  unsigned long long wait_timeout_ns = 300ull * 1000000000ull;
  std::set<esp_ctx_s*> ctxs;
  // hierarchical communication (reading R23): n = m machines x g
  // GPUs; the intra-machine phases run on `intra`, the compressed
  // inter-machine phase on `inter` (both owned)
  int hier_g = 0;                          // > 0: a hierarchical world
  esp_world_s* intra = nullptr;            // the g GPUs of this rank's machine
  esp_world_s* inter = nullptr;            // the m GPUs with this rank's local index
  std::vector<esp::HierPlan*> hplans;      // owned
};

struct esp_ctx_s {
  esp_world_s* w = nullptr;
  esp_compressor_cfg_t cfg{};
  int routine = 0;
  uint64_t tensor_id = 0;
  uint64_t N = 0;
  int P = 1;                         // partitions of the first compression
  std::vector<uint32_t> plo, phi, pk;
  uint32_t kpad = 0;                 // entries (sparse) or words (sign) per chunk
  size_t chunk_bytes = 0, payload_bytes = 0;
  // state (device), per local rank
  float* r = nullptr;                // nlocal * N
  float* lazy = nullptr;             // nlocal * P * 2
  float* r2 = nullptr;               // nlocal * r2_len   (second residual, R11)
  float* lazy2 = nullptr;            // nlocal * 2
  float* u = nullptr;                // nlocal * N: DGC momentum buffer (cfg.momentum != 0)
  // DGC / TOPK deferred EF zeroing records (k_dgc.cu), per local rank: the
  // 4096-element tiles of every partition of r (zrec) and of r2 (zrec2)
  uint16_t* zrec = nullptr;
  uint16_t* zrec2 = nullptr;
  uint32_t zcap = 0;                 // uint16 per tile record (32, 64 or 128)
  std::vector<size_t> zrec_part;     // partition p's first record inside a rank's block
  size_t zrec_stride = 0, zrec2_stride = 0;
  uint64_t r2_len = 0;
  uint64_t step = 0;
  uint64_t hash_base = 0;            // mix(mix(seed) ^ tensor_id)
  esp_ctx_s* inner = nullptr;        // hierarchical world: this rank's shard as a ctx of w->inter (owned)
  // esp_decompress: device tables of the last (pieces, out) seen, reused while
  // the caller passes the same buffers; staged through pinned memory
  struct DecCache {
    std::vector<const void*> pieces;
    float* out = nullptr;
    bool valid = false;
    unsigned char* d = nullptr;      // device tables
    size_t dcap = 0;
    unsigned char* h = nullptr;      // pinned staging (guarded by ev)
    size_t hcap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
    size_t off_seg = 0, off_units = 0, off_pp = 0, off_rt = 0, off_ps = 0;
    uint32_t nunits = 0;
    int njobs = 0;
    uint64_t step_uploaded = ~0ull;  // Randomk: step of the dyn word on the device
    float* acc = nullptr;            // accumulate mode: the aggregate before out += it
  } dec;
};

namespace esp {

// ---- collective layer -------------------------------------------------------
// Every call records per-rank bytes in w->counters with the cost-table
// conventions (see esp.h).  In the sim world, lr-indexed buffers are
// nlocal slices of `stride` bytes.
struct LocalBufs {
  unsigned char* base;
  size_t stride;      // bytes between local ranks
  unsigned char* at(int lr) const { return base + (size_t)lr * stride; }
};
void coll_allgather(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t bytes, cudaStream_t st);
void coll_alltoall(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t chunk, cudaStream_t st);
void coll_gather(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t bytes, cudaStream_t st);
void coll_broadcast(esp_world_s* w, LocalBufs buf, size_t bytes, cudaStream_t st);
void coll_allreduce_f32(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t count, cudaStream_t st);
void coll_reducescatter_f32(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t count, cudaStream_t st);
void coll_reduce_f32(esp_world_s* w, LocalBufs send, LocalBufs recv, size_t count, cudaStream_t st);
void coll_allgather_inplace_f32(esp_world_s* w, LocalBufs buf, size_t count_per_rank, cudaStream_t st);

// ---- plans ------------------------------------------------------------------
Plan* get_plan(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs);
Plan* find_plan(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs);   // nullptr if not cached
void drop_plans_with(esp_world_s* w, esp_ctx_s* c);
void execute_plan(Plan* p, float* const* grads, cudaStream_t st);
// the n worlds of a loopback group as ranks 0..n-1 on one GPU (plans[r] of world r)
void execute_loopback(const std::vector<Plan*>& plans, const std::vector<float* const*>& grads, cudaStream_t st);
// h1 only, copying each rank's payload to `payload` (esp_compress)
void execute_compress(Plan* p, const float* grad, void* payload, cudaStream_t st);
void clear_plans(esp_world_s* w);
void trim_plans(esp_world_s* w);   // evict least recently used plans down to w->plan_cap
// hierarchical worlds (hier.cu)
void execute_hier(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs, float* const* grads, cudaStream_t st);
void execute_hier_loopback(const std::vector<esp_world_s*>& ws, const std::vector<std::vector<esp_ctx_s*>>& ctxs,
                           const std::vector<float* const*>& grads, cudaStream_t st);
void clear_hier_plans(esp_world_s* w);
void drop_hier_plans_with(esp_world_s* w, esp_ctx_s* c);

}  // namespace esp

#define ESP_API_BEGIN try {
#define ESP_API_END                                  \
  }                                                  \
  catch (const ::esp::Fail& f) {                     \
    return f.st;                                     \
  }                                                  \
  catch (const std::bad_alloc&) {                    \
    ::esp::set_error("host out of memory");          \
    return ESP_ERR_OOM;                              \
  }                                                  \
  catch (...) {                                      \
    ::esp::set_error("unexpected exception");        \
    return ESP_ERR_STATE;                            \
  }                                                  \
  return ESP_OK;

