/*
 * esp.h — C ABI of the B200-native Espresso (arXiv 2205.14465) compressed
 * gradient-synchronisation hot path.
 *
 * What it computes (App. A): for each gradient
 * tensor of a data-parallel job, h1 = compression fused with its
 * error-feedback residual update (G5), then the chosen collective
 * routine ("The collective routines for synchronization"), then
 * h2 = fused decompression + aggregation of the n (or n^2) received pieces
 * ("fuses the decompression operations").  The per-tensor option is the
 * paper's compression option c_j restricted to flat
 * communication on GPU: a (compressor, ratio, routine) triple.
 *
 * Conventions
 *   - Every call returns esp_status_t; the library never aborts or throws.
 *     Argument errors are reported synchronously; asynchronous CUDA/NCCL errors
 *     surface on the next call or via esp_world_check().  esp_last_error()
 *     returns a thread-local message for the last failure.
 *   - All device work is enqueued on the caller's stream (cudaStream_t passed as
 *     void*; NULL = legacy default stream).  The library also uses one internal
 *     communication stream per world, joined back to the caller's stream with
 *     events before a call returns.
 *   - Ownership: the caller owns gradients, user payload buffers and streams;
 *     the library owns worlds, ctx state (EF residuals) and workspaces.
 *     Nothing is allocated on the hot path after the first call with a given
 *     tensor set (plans are cached).
 *   - Threading: one host thread per world at a time (an NCCL rule).
 *   - Gradients are contiguous fp32 device pointers, 4-byte aligned for
 *     esp_sync / esp_sync_many (16-byte aligned ones take the TMA fast path),
 *     16-byte aligned for esp_compress / esp_decompress buffers;
 *     numel < 2^31 (indices are uint32, reading R18) else ESP_ERR_TOO_LARGE.
 *   - Sim world: n virtual ranks on one GPU.  Every per-rank buffer argument is
 *     then n rank-major slices (rank r at offset r * slice) and collectives are
 *     device-to-device copies among the slices.
 *
 * Payload layouts (16-byte aligned sections; a tensor's payload is P equal-size
 * chunks, one per partition, P = n for Alltoall/Allgather else 1; see
 * esp_compressed_bytes):
 *   DGC / TOPK : uint32 idx[k_pad] then float val[k_pad]; idx relative to the
 *                partition start, ascending; padding idx = 0xFFFFFFFF, val = +0
 *   RANDOMK    : float val[k_pad] (indices regenerate from the seed, R5)
 *   EFSIGNSGD  : float scale, 12 pad bytes, uint32 words[w_pad] (bit l of word w
 *                is element 32w + l, LSB first, 1 <=> p >= 0; tail bits 0)
 *   ONEBIT     : float mean_neg, float mean_pos, 8 pad bytes, words as above
 *   NONE       : float values[numel]
 */
#ifndef ESP_H_
#define ESP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  ESP_OK = 0,
  ESP_ERR_INVALID_ARG = 1,  /* null pointer, bad enum, misaligned, wrong size */
  ESP_ERR_UNSUPPORTED = 2,  /* illegal (compressor, routine) pair */
  ESP_ERR_TOO_LARGE = 3,    /* numel >= 2^31 */
  ESP_ERR_CUDA = 4,
  ESP_ERR_NCCL = 5,
  ESP_ERR_OOM = 6,
  ESP_ERR_STATE = 7         /* object used with the wrong world / state blob */
} esp_status_t;

/* Compressors the paper evaluates (Randomk, DGC at 1%, EFSignSGD;
 * App. D figures: Onebit).  TOPK = DGC's exact result without the sampled
 * threshold accelerator (reading R3): every element enters the exact radix
 * select, the unsampled baseline DGC's threshold speeds up.  NONE =
 * uncompressed fp32. */
typedef enum {
  ESP_NONE = 0, ESP_RANDOMK = 1, ESP_DGC = 2, ESP_TOPK = 3, ESP_EFSIGNSGD = 4, ESP_ONEBIT = 5
} esp_kind_t;

/* Routines of P:1057-1070 (flat communication, root = rank 0, reading R17). */
typedef enum {
  ESP_ALLREDUCE = 0,
  ESP_ALLGATHER = 1,
  ESP_ALLTOALL_ALLGATHER = 2,     /* sparse: process 1; quantized: process 2 */
  ESP_GATHER_BROADCAST = 3,       /* sparse: process 1; quantized: process 2 */
  ESP_REDUCESCATTER_ALLGATHER = 4,
  ESP_REDUCE_BROADCAST = 5
} esp_routine_t;

typedef enum { ESP_MEAN = 0, ESP_SUM = 1 } esp_reduce_t;  /* reading R9 */

typedef struct {
  int32_t kind;                   /* esp_kind_t */
  int32_t error_feedback;         /* 1: e <- (g+e) - C(g+e) (G5) */
  double ratio;                   /* rho in (0, 1]; k = min(N, max(1, ceil(rho*N))) (R1) */
  uint64_t seed;                  /* Randomk hash seed */
  int32_t randomk_shared_indices; /* 1: same indices on every rank => allreducible (R5) */
  int32_t reduce;                 /* esp_reduce_t */
  /* Alltoall/Allgather and Gather/Broadcast (App. A, reading R19):
   * 1 = forward the first compression's chunks (decompress n^2 resp. n pieces),
   * 2 = decompress + aggregate + recompress mid-scheme with a second residual
   * (alpha = 1/n resp. 1); 0 = the cost table's choice ("the first process for
   * sparse tensors and the second process for quantized tensors").
   * Ignored by the other routines; other values -> ESP_ERR_INVALID_ARG. */
  int32_t process;
  /* DGC / TOPK momentum correction with momentum factor masking (the DGC
   * algorithm cited at P:828, reading R20), m in [0, 1):
   * u <- fl(fl(m*u) + g), v <- fl(v + u), select top-k of v, transmit v[sel],
   * v[sel] <- 0, u[sel] <- 0.  0 = off (plain error feedback, R4).  Requires
   * error_feedback = 1 and kind DGC or TOPK, else ESP_ERR_INVALID_ARG. */
  double momentum;
  /* DGC sampled threshold (the DGC algorithm cited at P:828, SURVEY.md 8f
   * NEXT-2, reading R22).  The sample of a segment of N > 4096 elements is S
   * strata of 8 consecutive elements at hashed offsets; dgc_sample_rate = 0
   * gives S = 512 (4096 samples), else S = ceil(rate * N / 8) clipped to
   * [1, 512].  dgc_approx = 0 (exact, the default): the threshold only
   * accelerates and exactly the top-k is selected (R3).  dgc_approx = 1
   * (approximate-count mode, DGC's own selection): every element whose key
   * passes the threshold of the round(rho * s)-th largest sampled key is
   * selected, the exact top-k of them if more than k pass; fewer than k entries
   * are then sent and the rest of the chunk is padding.  DGC only, else
   * ESP_ERR_INVALID_ARG (as is a rate outside [0, 1]). */
  int32_t dgc_approx;
  double dgc_sample_rate;
} esp_compressor_cfg_t;

typedef struct esp_world_s* esp_world_t;
typedef struct esp_ctx_s* esp_ctx_t;

/* Counters of one world (reset by esp_world_reset_counters).  Byte counts are
 * per rank (per virtual rank 0 in a sim world) and follow the cost-table
 * conventions of P:52-117: Allgather receives (n-1)M, Alltoall (n-1)M/n, ring
 * Allreduce 2(n-1)M/n, Gather (n-1)M at the root, Broadcast X at a non-root. */
enum { ESP_OP_ALLREDUCE = 0, ESP_OP_ALLGATHER, ESP_OP_ALLTOALL, ESP_OP_GATHER,
       ESP_OP_BROADCAST, ESP_OP_REDUCESCATTER, ESP_OP_REDUCE, ESP_NUM_OPS };
typedef struct {
  uint64_t calls[ESP_NUM_OPS];
  uint64_t sent[ESP_NUM_OPS];
  uint64_t recv[ESP_NUM_OPS];
  uint64_t h1_calls;      /* compress applications on the critical rank */
  uint64_t h2_pieces;     /* decompressed pieces on the critical rank */
  uint64_t pushed;        /* bytes this rank actually stored into peers' memory over
                             NVLink (fused collectives; the cost-table figures above
                             are logical volumes) */
} esp_counters_t;

/* Per-phase device times of the last esp_sync / esp_sync_many (ms, CUDA events;
 * only when timing is enabled with esp_world_set_timing). */
typedef struct {
  float total_ms, h1_ms, comm_ms, mid_ms, h2_ms;
} esp_timing_t;

/* ---- world ---------------------------------------------------------------
 * esp_get_nccl_unique_id: writes 128 bytes (ncclUniqueId) to out128 (host).
 * esp_world_create_nccl: one process per GPU; id128 identical on all ranks;
 *   creates and owns an ncclComm_t on cuda_dev.
 * esp_world_create_sim: nranks virtual ranks on cuda_dev (config 1).
 */
esp_status_t esp_get_nccl_unique_id(void* out128);
esp_status_t esp_world_create_nccl(const void* id128, int nranks, int rank, int cuda_dev,
                                   esp_world_t* out);
esp_status_t esp_world_create_sim(int nranks, int cuda_dev, esp_world_t* out);
/* Loopback group (tests): nranks worlds in this process on one GPU, out[r]
 * acting as rank r of an nranks-rank job with the fused (byte-moving)
 * collectives of a real multi-GPU run -- the same job tables, slot layouts,
 * arrival counters and call parities -- over plain device pointers instead of
 * CUDA IPC.  Synchronised only through esp_sync_many_loopback, which runs
 * every rank's kernels on one stream in dependency order (no kernel waits for
 * a later one).  NCCL-reduced buckets (NONE, Randomk Allreduce) are
 * ESP_ERR_UNSUPPORTED here.  Each world is destroyed with esp_world_destroy. */
esp_status_t esp_world_create_loopback(int nranks, int cuda_dev, esp_world_t* out /* [nranks] */);
/* Hierarchical communication (aggregate within each machine, then
 * across machines, then within each machine again; SURVEY.md 8f NEXT-4,
 * reading R23).  The parent's n ranks form m = n / group "machines" of group
 * consecutive ranks (emulated on one NVLink box).  On the returned world a
 * ctx (compressed kinds; routine = the inter-machine routine: ALLGATHER,
 * ALLTOALL_ALLGATHER or GATHER_BROADCAST) synchronises its tensor in three
 * phases: an uncompressed intra-machine Reduce-scatter into group shards
 * (R10 partitions; shard i on local rank i, the machine's mean for MEAN), the
 * compressed inter-machine routine of each shard among the m ranks holding
 * it (error feedback per rank and shard), and an intra-machine Allgather of
 * the shards.  The parent stays the caller's; esp_world_create_hier is
 * collective over it (two ncclCommSplit).  esp_world_create_loopback_hier:
 * the same as a loopback group on one GPU (tests; esp_sync_many_loopback).
 * ctx state (get/set_state) is that of the rank's shard. */
esp_status_t esp_world_create_hier(esp_world_t parent, int group, esp_world_t* out);
esp_status_t esp_world_create_loopback_hier(int nranks, int group, int cuda_dev, esp_world_t* out /* [nranks] */);
esp_status_t esp_world_destroy(esp_world_t w);
esp_status_t esp_world_check(esp_world_t w);   /* async CUDA/NCCL errors */
esp_status_t esp_world_info(esp_world_t w, int* nranks, int* rank, int* nlocal);
esp_status_t esp_world_counters(esp_world_t w, esp_counters_t* out);
/* counters of local rank lr (sim world: virtual rank lr) */
esp_status_t esp_world_counters_local(esp_world_t w, int lr, esp_counters_t* out);
esp_status_t esp_world_reset_counters(esp_world_t w);
esp_status_t esp_world_set_timing(esp_world_t w, int enable);
esp_status_t esp_last_timing(esp_world_t w, esp_timing_t* out);
/* Max elements per bucket of esp_sync_many (0 = library default).  Smaller
 * buckets pipeline h1 / comm / h2 across buckets (a9). */
esp_status_t esp_world_set_bucket_elems(esp_world_t w, uint64_t elems);
/* Dominant-kernel probe (roofline evidence): while enabled, CUDA events are
 * recorded on the launching stream around the streaming h1 kernel of every
 * bucket (DGC/TOPK: the fused g + r pass; Randomk/sign: their h1 kernel; NONE:
 * the pack copy).  esp_probe_read waits for them and returns the summed device
 * time (ms), the number of probed launches and the algorithmic HBM bytes those
 * launches had to move (12 B/elem with EF, +1/8 B/elem of sign bits), then
 * clears the record. */
esp_status_t esp_world_set_probe(esp_world_t w, int enable);
/* Fused collectives (n > 1): a rank waits for its peers' payloads on the GPU.
 * If a payload has not arrived after `seconds` of wall time (default 300), the
 * wait gives up, the call's output is invalid, and esp_world_check plus every
 * later esp_sync / esp_sync_many return ESP_ERR_NCCL (the world is unusable). */
esp_status_t esp_world_set_timeout(esp_world_t w, double seconds);
/* Execution plans (bucketing, device tables, buffers) are cached per tensor
 * list.  set_plan_cache bounds the cache (least recently used plans are freed;
 * default 64); drop_plans frees all of them (e.g. when a training framework
 * rebuilds its gradient buckets).  Every rank must make the same calls. */
esp_status_t esp_world_set_plan_cache(esp_world_t w, int max_plans);
/* NVLS multicast for the fused Allgather (NVSwitch replicates one store of a
 * rank's payload into every GPU's receive buffer): -1 auto (default; on when
 * every rank's GPU supports multicast and n >= 3), 0 off (unicast peer
 * copies), 1 on whenever supported.  Same value on every rank; frees the
 * world's cached plans. */
esp_status_t esp_world_set_multicast(esp_world_t w, int mode);
esp_status_t esp_world_drop_plans(esp_world_t w);
esp_status_t esp_probe_read(esp_world_t w, double* ms, uint64_t* launches, uint64_t* bytes);

/* ---- ctx: one tensor's option + EF state ----------------------------------
 * Validates the (compressor, routine) pair: NONE -> {ALLREDUCE,
 * REDUCESCATTER_ALLGATHER, REDUCE_BROADCAST}; DGC/TOPK/EFSIGNSGD/ONEBIT ->
 * {ALLGATHER, ALLTOALL_ALLGATHER, GATHER_BROADCAST}; RANDOMK -> those plus
 * ALLREDUCE when randomk_shared_indices;
 * anything else -> ESP_ERR_UNSUPPORTED.  Allocates the residual(s) (zeroed)
 * and the workspace for every local rank of the world.
 */
esp_status_t esp_ctx_create(esp_world_t w, const esp_compressor_cfg_t* cfg, int routine,
                            uint64_t tensor_id, size_t numel, esp_ctx_t* out);
esp_status_t esp_ctx_destroy(esp_ctx_t c);
/* Bytes of one rank's first-compression payload (P chunks). */
esp_status_t esp_ctx_payload_bytes(esp_ctx_t c, size_t* out);
/* EF state blob (host memory): header {uint64 magic, step, numel, r2_len,
 * nlocal} then per local rank: float r[numel], float r2[r2_len].  r / r2 are
 * the TRUE residuals (materialised from the lazy representation).  Pass
 * host_buf = NULL to query the size.  set_state restores a blob (synchronous). */
esp_status_t esp_ctx_get_state(esp_ctx_t c, void* host_buf, size_t* nbytes);
esp_status_t esp_ctx_set_state(esp_ctx_t c, const void* host_buf, size_t nbytes);
/* The momentum buffer u of a ctx with cfg.momentum != 0: `count` must be
 * nlocal * numel floats (host memory, rank-major in a sim world).
 * ESP_ERR_STATE if the ctx has no momentum buffer. */
esp_status_t esp_ctx_get_momentum(esp_ctx_t c, float* host, size_t count);
esp_status_t esp_ctx_set_momentum(esp_ctx_t c, const float* host, size_t count);

/* ---- h1 / h2 ----------------------------------------------------------------
 * esp_compress: EF-fused compression of one rank's tensor (every local rank in a
 * sim world).  payload: esp_ctx_payload_bytes bytes per rank, caller-owned.
 * Advances the ctx step counter (Randomk draws).
 * esp_decompress: agg[numel] = reduce(sum over pieces in order of decompress(
 * pieces[i])) — rank-order fp32 sum from +0.0f, then / npieces for MEAN;
 * accumulate = 0: out := agg; accumulate = 1: out[i] := fl(out[i] + agg[i])
 * for every i (through a per-ctx temporary).
 * pieces: npieces device pointers (host array) to full payloads of this ctx.
 */
esp_status_t esp_compress(esp_ctx_t c, const float* grad, void* payload, void* stream);
esp_status_t esp_decompress(esp_ctx_t c, const void* const* pieces, int npieces, float* out,
                            int accumulate, void* stream);

/* ---- sync ---------------------------------------------------------------------
 * h1 -> routine -> h2.  grad_inout := the aggregated gradient on every rank.
 * esp_sync_many runs a per-tensor strategy over a tensor set with bucketing
 * (one multi-tensor h1 launch, one collective and one h2 launch per bucket).
 */
esp_status_t esp_sync(esp_world_t w, esp_ctx_t c, float* grad_inout, void* stream);
esp_status_t esp_sync_many(esp_world_t w, const esp_ctx_t* ctxs, float* const* grads,
                           int ntensors, void* stream);
/* esp_sync_many for every rank of a loopback group: ctxs and grads are
 * [nranks][ntensors] (rank-major), ctxs[r][.] created on worlds[r]. */
esp_status_t esp_sync_many_loopback(const esp_world_t* worlds, int nranks, const esp_ctx_t* ctxs,
                                    float* const* grads, int ntensors, void* stream);

/* ---- sizes / cost table ----------------------------------------------
 * esp_compressed_bytes: bytes of one rank's payload for numel elements split
 * into nparts partitions (R10).
 * esp_wire_bytes: the communication volume of a routine for a tensor type,
 *   per rank on the critical path, for a payload (or, uncompressed, a tensor)
 *   of M bytes over n ranks -- the cost table's communication column times B
 *   (S:126 for the uncompressed pairs).  tensor_type:
 *   ESP_TT_ALLREDUCIBLE (uncompressed fp32, or Randomk values with shared
 *   indices), ESP_TT_SPARSE (first process of a divisible routine, P:70-76 /
 *   P:97-103; any compressed payload for Allgather), ESP_TT_QUANTIZED (second
 *   process, P:78-87 / P:105-115).  The table models every row as one volume
 *   over a full-duplex link, so *sent == *recv.  Volumes:
 *     ALLREDUCE, allreducible            2(n-1)M/n
 *     REDUCESCATTER_ALLGATHER, allred.   (n-1)M/n + (n-1)M/n
 *     REDUCE_BROADCAST, allreducible     (n-1)M + M
 *     ALLGATHER, sparse or quantized     (n-1)M
 *     ALLTOALL_ALLGATHER, sparse         (n^2-1)M/n;  quantized 2(n-1)M/n (R13)
 *     GATHER_BROADCAST, sparse           (2n-1)M;     quantized nM
 *   0 for n = 1.  Any other (routine, type) pair -> ESP_ERR_UNSUPPORTED.
 * esp_model_time: that volume / B seconds (B in bytes/s).
 */
enum { ESP_TT_ALLREDUCIBLE = 0, ESP_TT_SPARSE = 1, ESP_TT_QUANTIZED = 2 };
esp_status_t esp_compressed_bytes(const esp_compressor_cfg_t* cfg, size_t numel, int nparts,
                                  size_t* out);
esp_status_t esp_wire_bytes(int routine, int tensor_type, double M, int n, double* sent, double* recv);
esp_status_t esp_model_time(int routine, int tensor_type, double M, int n, double B, double* out_seconds);

/* ---- strategy selection (App. A; Algorithm 1
 * P:1299-1361; readings R15, R21) -----------------------------------------------
 * esp_curve_t: a measured cost curve, n samples (input bytes, seconds) with
 *   strictly increasing bytes ("profiled ... 2^10, 2^11, ..., 2^30", P:27-29;
 *   tools/sweep.py).  esp_curve_eval: log-log piecewise-linear interpolation,
 *   clamped to the first sample below it, the last segment's slope above the
 *   last sample ("curve fitting").  ESP_ERR_INVALID_ARG on an empty or
 *   non-increasing curve or a non-positive sample.
 * esp_option_t: one candidate compression option of a tensor (the paper's c_j
 *   restricted to GPU + flat communication): compressor cfg, routine, and the
 *   h1 / h2 curves of that compressor (ignored for NONE).
 * esp_option_time: predicted synchronisation time of one tensor of numel fp32
 *   over n ranks at B bytes/s: the cost table's communication column for the
 *   option's row with M = its payload bytes, plus the table's compression
 *   column with h1(.) / h2(.) evaluated at the input bytes of each application
 *   (h1(M) = h1 at 4 numel bytes, h1(M/n) and h2(M/n) at 4 numel / n); NONE has
 *   no compression time.  ESP_ERR_UNSUPPORTED for an illegal pair.
 * esp_select_option: Algorithm 1's GetBestOption for one tensor with no
 *   computation to overlap (R21): the argmin of esp_option_time over the
 *   candidates (ties: lowest index); *best = its index.
 */
typedef struct {
  const double* bytes;
  const double* seconds;
  int32_t n;
} esp_curve_t;
typedef struct {
  esp_compressor_cfg_t cfg;
  int32_t routine;
  esp_curve_t h1, h2;
} esp_option_t;
esp_status_t esp_curve_eval(const esp_curve_t* c, double bytes, double* out_seconds);
esp_status_t esp_option_time(const esp_option_t* opt, size_t numel, int n, double B, double* out_seconds);
esp_status_t esp_select_option(const esp_option_t* opts, int nopt, size_t numel, int n, double B, int* best,
                               double* out_seconds);

/* ---- diagnostics --------------------------------------------------------------- */
const char* esp_status_string(esp_status_t s);
const char* esp_last_error(void);
uint64_t esp_launch_count(void);   /* kernels this library launched (process total) */
const char* esp_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* ESP_H_ */
