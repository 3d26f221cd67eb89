// Execution plans: bucketing of a tensor set by (compressor, routine), the
// device work tables of every kernel, the buffers of every collective phase,
// and the pipelined executor ("Multiple CUDA
// streams are used to overlap the computation, communication, and
// compression").  A plan is built once per tensor list and cached on the world;
// a call then costs one 16-byte-per-tensor async H2D copy of the gradient
// pointers and step counters plus the kernel/collective launches.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>

#include "esp_internal.h"
#include "esp_kernels.h"
#include "mcast.h"

namespace esp {

struct Bucket {
  int kind = 0, routine = 0, reduce = 0;
  int proc = 1;                // process of a divisible routine (R19)
  double momentum = 0.0;       // DGC momentum correction factor (R20)
  bool ef = true;              // error feedback (all tensors of a bucket agree)
  bool p2 = false;             // mid-scheme decompress-aggregate-recompress (a7)
  std::vector<int> tens;      // indices into Plan::ctxs
  int P = 1;
  size_t slot = 0;            // bytes of one slot = sum of the tensors' chunks
  std::vector<size_t> coff;   // chunk offset of each tensor within a slot
  size_t none_count = 0;      // NONE: floats in the packed slot (padded to n)
  uint64_t none_bytes = 0;    // NONE: logical bytes (sum of 4 N_t) for the counters
  LocalBufs send{}, recv1{}, recv2{}, mid{};
  // tables (device) and sizes
  SegH1* h1 = nullptr; int nh1 = 0;
  uint32_t* h1_units = nullptr; int nh1_units = 0;
  uint32_t* h1_groups = nullptr; int nh1_groups = 0;
  SegH1* a7 = nullptr; int na7 = 0;
  uint32_t* a7_units = nullptr; int na7_units = 0;
  const unsigned char** a7_pieces = nullptr;
  // a7 of a sparse compressor (process 2): h2 of the n chunks into a dense
  // temporary (a7h2), then the compressor's h1 on it with r = r2 (a7)
  uint32_t* a7_groups = nullptr; int na7_groups = 0;
  SegH2* a7h2 = nullptr; int na7h2 = 0;
  uint32_t* a7h2_units = nullptr; int na7h2_units = 0;
  uint32_t* a7h2_rankterms = nullptr;
  uint4* a7h2_off_jobs = nullptr; int na7h2_off_jobs = 0;
  uint64_t* a7ptr = nullptr;   // device [nlocal]: base of each local rank's temporary
  LocalBufs a7tmp{};
  SegH2* h2 = nullptr; int nh2 = 0;
  uint32_t* h2_units = nullptr; int nh2_units = 0;
  const unsigned char** h2_pieces = nullptr;
  uint32_t* h2_rankterms = nullptr;
  uint4* h2_off_jobs = nullptr; int nh2_off_jobs = 0;
  bool h2_dense = false;     // sparse h2: the CTA-tile kernel (launch_h2_sparse)
  uint32_t rpg_cap = kRunsPerGroup;   // DGC finalize group length cap (dgc_rpg_cap)
  bool a7h2_dense = false;
  int h2_max_pieces = 0;
  uint32_t h1_max_len = 0, a7_max_len = 0;   // longest h1 / a7 segment
  bool small = false;          // DGC: every h1 segment has <= kSample elements (one-kernel h1)
  bool onchip = false;         // DGC: the bucket fits on chip (dgc_mid_kernel, one kernel)
  uint32_t onchip_tpc = 0;     //   tiles per CTA
  int onchip_grid = 0;         //   CTAs (<= #SMs, all co-resident)
  cudaEvent_t ev_h1 = nullptr, ev_comm = nullptr, ev_stream = nullptr;
  uint64_t h1_calls = 0, h2_pieces_count = 0;   // per tensor-rank counters
  uint64_t h1_bytes = 0;      // algorithmic HBM bytes of the streaming h1 kernel
  // ---- compression fused with the collective over NVLink peer memory
  // (DESIGN.md 9): the producers (DGC write, sign h1 /
  // a7) write their payload locally, then push_kernel copies each slot
  // straight to its final place in the receiving ranks' buffers
  // (double-buffered by call parity) and bumps their arrival counters; the
  // consumer starts after a wait kernel has seen this call's arrivals.
  //   phase 1 = send -> recv1 (Allgather, Alltoall, Gather) or recv2 (sparse
  //             Alltoall/Allgather: chunk (part, src) goes straight to its
  //             final place on every rank, the forwarding hop disappears)
  //   phase 2 = stage (a7's output) -> recv2 (quantized Alltoall/Allgather)
  //             or mid (quantized Gather/Broadcast, from the root)
  bool fused = false;
  size_t dst1_off = 0, dst1_par = 0, dst1_slot = 0;   // phase-1 destination: off + par * par_stride + src * slot
  size_t dst2_off = 0, dst2_par = 0, dst2_slot = 0;   // phase-2 destination
  // arrival counters, one per (phase, call parity): [2 * phase + parity].  A
  // peer's call-(t+2) arrivals can only follow its call-(t+1) consumers,
  // which follow every call-t push of that peer in stream order, so a
  // parity's counter never runs ahead of a call it has not completed
  size_t cnt_off = 0;
  uint64_t target1 = 0, target2 = 0;            // arrivals per call
  LocalBufs stage{};
  PushJob* push1 = nullptr; int npush1 = 0;
  PushJob* push2 = nullptr; int npush2 = 0;
  uint64_t push1_bytes = 0, push2_bytes = 0, push2_odd_bytes = 0;   // bytes moved per call
  // NVLS multicast (Allgather; mcast.cu): my slot's jobs once, to the
  // multicast alias of every rank's receive buffer in the plan's region
  bool mc = false;
  PushJob* push1_mc = nullptr; int npush1_mc = 0;
  unsigned char* mc_recv = nullptr;             // multicast alias of this bucket's [2][n][S] receive buffer
  unsigned long long* mc_cnt = nullptr;         // multicast alias of the bucket's 4 counters
  int npiece_ptrs = 0;                          // entries of h2_pieces (and h2_pieces_odd)
  // process-1 Gather/Broadcast: the root forwards all n payloads; its jobs read
  // from anywhere in its arena (own payload: send, the others: recv1 of the
  // call's parity), so there is one table per parity and src = arena base
  PushJob* push2_odd = nullptr;
  bool push2_arena = false;
  size_t send_off = 0;
  const unsigned char** h2_pieces_odd = nullptr;   // h2 pieces of the parity-1 buffers
  const unsigned char** a7_pieces_odd = nullptr;
  unsigned char** dsts = nullptr;               // device [2][n]: my phase-1 slot in every rank's buffer
  unsigned char** dsts2 = nullptr;              // device [2][n]: my phase-2 slot
  unsigned long long** cnts = nullptr;          // device [2][n]: every rank's phase-1 counter per parity
  unsigned long long** cnts2 = nullptr;         // device [2][n]: every rank's phase-2 counter per parity
  unsigned long long* my_cnt = nullptr;         // my 4 counters [2 * phase + parity]
  uint64_t epoch = 0;
};

// A CUDA graph of one call's device work (every launch, copy and memset after
// the gradient-pointer upload), captured on the first call and replayed after:
// one cudaGraphLaunch instead of a dozen API calls per call (the per-call
// "constant overhead to launch GPU kernels").  Only plans whose work
// never changes between calls are graphed (no fused collective: those use
// call-parity buffers and targets); the host-side counters a call adds are
// recorded at capture and re-added on every replay.
struct GraphCache {
  cudaGraphExec_t exec = nullptr;
  int key = -1;                          // launch-time inputs baked into the graph (test hooks)
  uint64_t launches = 0;                 // kernels per replay (esp_launch_count)
  std::vector<esp_counters_t> delta;     // per local rank
  ~GraphCache() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

struct Plan {
  esp_world_s* w = nullptr;
  GraphCache g_sync, g_compress;
  std::vector<esp_ctx_s*> ctxs;
  std::vector<Bucket> buckets;
  Arena arena;
  unsigned char* zero = nullptr;
  size_t zero_bytes = 0;
  uint64_t* dyn_dev = nullptr;
  // dyn words staged through a ring of pinned slots: the host waits only for the
  // copy of kDynSlots calls ago, so it can run ahead of the GPU
  static constexpr int kDynSlots = 16;
  uint64_t* dyn_host = nullptr;        // kDynSlots x 2 * nctxs
  cudaEvent_t dyn_ev[kDynSlots] = {};
  bool dyn_pending[kDynSlots] = {};
  int dyn_slot = 0;
  bool needs_step = false;             // some kernel reads the step words (Randomk)
  std::vector<const float*> dyn_last;  // gradient pointers of the last upload
  bool peers_ready = false;             // fused buckets: peer arenas opened (first collective call)
  std::unique_ptr<McRegion> mcr;        // NVLS multicast region of the plan's Allgather buckets
  std::vector<void*> peer_bases;        // IPC-opened arenas of the other ranks
  ~Plan() {
    for (void* pb : peer_bases)
      if (pb) cudaIpcCloseMemHandle(pb);
    for (auto& b : buckets) {
      if (b.ev_h1) cudaEventDestroy(b.ev_h1);
      if (b.ev_comm) cudaEventDestroy(b.ev_comm);
      if (b.ev_stream) cudaEventDestroy(b.ev_stream);
      if (b.dsts) cudaFree(b.dsts);
      if (b.dsts2) cudaFree(b.dsts2);
      if (b.cnts) cudaFree(b.cnts);
      if (b.cnts2) cudaFree(b.cnts2);
    }
    for (auto& e : dyn_ev)
      if (e) cudaEventDestroy(e);
    if (dyn_host) cudaFreeHost(dyn_host);
  }
};

static int grank(esp_world_s* w, int lr) { return w->sim ? lr : w->rank; }

// ------------------------------------------------------------------ layout
// Two passes over the same code: the first reserves arena offsets to size the
// single cudaMalloc, the second fills host tables with real pointers.
struct Layout {
  Plan& p;
  bool commit;
  size_t reserve(size_t bytes) { return p.arena.reserve(bytes); }
  template <class T>
  T* ptr(size_t off) { return commit ? reinterpret_cast<T*>(p.arena.base + off) : nullptr; }
};

struct HostTables {
  std::vector<SegH1> h1, a7;
  std::vector<uint32_t> h1_units, h1_groups, a7_units, a7_groups, h2_units, a7h2_units, a7h2_rankterms;
  std::vector<SegH2> a7h2;
  std::vector<uint4> a7h2_off_jobs;
  std::vector<SegH2> h2;
  std::vector<const unsigned char*> a7_pieces, a7_pieces_odd, h2_pieces, h2_pieces_odd;
  std::vector<uint32_t> rankterms;
  std::vector<uint4> off_jobs;
  std::vector<PushJob> push1, push2, push2_odd, push1_mc;
};

static bool fused_allgather_enabled() {
  static const bool on = [] {
    const char* e = getenv("ESP_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

// push jobs: [src_off, src_off + bytes) -> destination d at dst_off, in kPushChunk pieces
static void add_push(std::vector<PushJob>& v, size_t src_off, size_t dst_off, size_t bytes, int d) {
  for (size_t c = 0; c < bytes; c += kPushChunk)
    v.push_back(PushJob{src_off + c, dst_off + c, (uint32_t)std::min<size_t>(kPushChunk, bytes - c), (uint32_t)d});
}

// ESP_DGC_PATH=chain (test hook, read when a plan is built): DGC / TOPK h1 of
// buckets that fit on chip takes the sample / stream / finalize chain instead
// of dgc_mid_kernel, so that both paths stay covered by the parity tests
static bool dgc_mid_enabled() {
  const char* e = getenv("ESP_DGC_PATH");
  return !(e && strcmp(e, "chain") == 0);
}

// DGC sampler strata of a segment (reading R22): 512 (4096 samples) by
// default, else ceil(rate * n / 8) clipped to [1, 512]
static uint16_t dgc_strata(uint64_t n, double rate) {
  if (rate <= 0.0) return (uint16_t)(kSample / 8);
  const double c = std::ceil(rate * (double)n / 8.0);
  return (uint16_t)(c < 1.0 ? 1.0 : (c > kSample / 8 ? kSample / 8 : c));
}

// DGC finalize group length (runs) of a segment: the largest power of two in
// [8, 128] whose expected candidate count stays within 16 refine batches
// (2048; measured: 8-run groups at 1% made GPT-2's refine + write 180 us --
// tens of thousands of groups, a long look-back):
// candidates per 512-element run ~ 512 x (sampled rank / sample size) when
// sampled, ~ 512 k / n for a whole-segment sample, ~ 1024 k / n for TOPK
// (the k-th key's 11-bit bin and above)
static uint32_t dgc_rpg(uint64_t len, uint32_t k, const esp_compressor_cfg_t& cfg, uint32_t cap) {
  double frac;
  if (cfg.kind == ESP_TOPK) {
    frac = 2.0 * k / (double)len;
  } else if (len <= (uint64_t)kSample) {
    frac = (double)k / (double)len;
  } else {
    const double s = 8.0 * dgc_strata(len, cfg.dgc_sample_rate), rs = cfg.ratio * s;
    double need = cfg.dgc_approx ? std::floor(rs + 0.5) : std::ceil(rs + 4.0 * std::sqrt(rs));
    need = need < 1.0 ? 1.0 : (need > s ? s : need);
    frac = need / s;
  }
  const double c_run = (double)kRun * (frac > 1.0 ? 1.0 : frac);
  uint32_t rpg = cap;
  while (rpg > 8 && rpg * c_run > 2048.0) rpg /= 2;
  return rpg;
}

static void fill_unit_table(std::vector<uint32_t>& units, uint32_t seg, uint32_t count) {
  for (uint32_t i = 0; i < count; ++i) units.push_back(seg);
}

// Slot layout and every buffer a peer may address (send, receive, mid, stage,
// arrival counters): reserved for all buckets FIRST, before anything whose
// size depends on the rank (a7 workspaces exist on owners only), so that the
// offsets inside the arena are identical on every rank (fused collectives
// address a peer's buffer as its arena base + the same offset).
static void layout_buffers(Layout& L, Bucket& b, HostTables& T) {
  Plan& p = L.p;
  esp_world_s* w = p.w;
  const int n = w->nranks, nl = w->nlocal;
  const bool none = b.kind == ESP_NONE;
  const bool dgc = b.kind == ESP_DGC || b.kind == ESP_TOPK;
  const bool quant = is_quant(b.kind);
  const bool divis = b.routine == ESP_ALLTOALL_ALLGATHER || b.routine == ESP_GATHER_BROADCAST;
  const bool p2 = !none && divis && b.proc == 2;   // mid-scheme recompression (a7)
  b.p2 = p2;
  // ---- slot layout
  b.coff.clear();
  b.slot = 0;
  if (none) {
    for (int t : b.tens) {
      b.coff.push_back(b.slot);
      b.slot += round_up(4 * p.ctxs[t]->N, 16);
    }
    b.none_bytes = 0;
    for (int t : b.tens) b.none_bytes += 4 * p.ctxs[t]->N;
    b.none_count = round_up(b.slot / 4, (size_t)n * 4);
    b.slot = b.none_count * 4;
  } else {
    for (int t : b.tens) {
      b.coff.push_back(b.slot);
      b.slot += round_up(p.ctxs[t]->chunk_bytes, 16);
    }
  }
  b.P = none ? 1 : p.ctxs[b.tens[0]]->P;
  const size_t S = b.slot;

  // ---- buffers (per local rank)
  auto bufs = [&](LocalBufs& lb, size_t per_rank) {
    size_t stride = round_up(per_rank, 256);
    size_t off = L.reserve(stride * nl);
    lb = LocalBufs{L.ptr<unsigned char>(off), stride};
    return off;
  };
  b.fused = fused_allgather_enabled() && !w->sim && n > 1 && !none &&
            (b.routine == ESP_ALLGATHER || b.routine == ESP_ALLTOALL_ALLGATHER ||
             b.routine == ESP_GATHER_BROADCAST);
  // (the fused producers write peers directly; the send buffer still serves esp_compress)
  b.send_off = bufs(b.send, b.P * S);
  // one real rank: every collective is the identity, so the receive buffers
  // alias the send/mid buffers and the collectives move nothing
  const bool solo = !w->sim && n == 1;
  if (solo) {
    b.recv1 = b.send;
    if (p2) {
      bufs(b.mid, S);
      b.recv2 = b.mid;
    } else {
      b.recv2 = b.send;
    }
  } else if (b.fused) {
    // two call-parity copies of every receive buffer; identical arena layouts on
    // every rank, so a peer's buffer is its arena base + the same offset
    b.cnt_off = L.reserve(256);
    if (b.routine == ESP_ALLGATHER) {
      b.dst1_off = bufs(b.recv1, 2 * n * S);
      b.dst1_par = (size_t)n * S;
      b.dst1_slot = S;
    } else if (b.routine == ESP_ALLTOALL_ALLGATHER && !p2) {   // process 1
      b.dst1_off = bufs(b.recv2, 2 * (size_t)n * n * S);
      b.dst1_par = (size_t)n * n * S;
      b.dst1_slot = S;
    } else if (b.routine == ESP_ALLTOALL_ALLGATHER) {   // process 2
      b.dst1_off = bufs(b.recv1, 2 * n * S);
      b.dst1_par = (size_t)n * S;
      b.dst1_slot = S;
      b.dst2_off = bufs(b.recv2, 2 * n * S);
      b.dst2_par = (size_t)n * S;
      b.dst2_slot = S;
    } else if (!p2) {                                   // Gather/Broadcast, process 1
      b.dst1_off = bufs(b.recv1, 2 * n * S);            // phase 1: every payload into the root's slot [src]
      b.dst1_par = (size_t)n * S;
      b.dst1_slot = S;
      b.dst2_off = b.dst1_off;                          // phase 2: the root's n payloads into every
      b.dst2_par = (size_t)n * S;                       // rank's recv1 (slot offsets in the jobs)
      b.dst2_slot = 0;
    } else {                                            // Gather/Broadcast, process 2
      b.dst1_off = bufs(b.recv1, 2 * n * S);
      b.dst1_par = (size_t)n * S;
      b.dst1_slot = S;
      b.dst2_off = bufs(b.mid, 2 * S);
      b.dst2_par = S;
      b.dst2_slot = 0;
    }
    {
      // jobs and arrivals per call (J jobs per slot)
      const uint64_t J = div_up(S, kPushChunk);
      const bool root = w->rank == 0;
      if (p2) bufs(b.stage, S);   // a7's local output
      // (no self copies: a rank reads its own chunks from the local source)
      const int me = w->rank;
      switch (b.routine) {
        case ESP_ALLGATHER:
          for (int d = 0; d < n; ++d)
            if (d != me) add_push(T.push1, 0, 0, S, d);
          add_push(T.push1_mc, 0, 0, S, 0);   // multicast: my slot once (open_peers decides)
          b.target1 = (n - 1) * J;
          break;
        case ESP_ALLTOALL_ALLGATHER:
          if (!p2) {
            for (int d = 0; d < n; ++d)
              for (int part = 0; part < b.P && d != me; ++part)
                add_push(T.push1, (size_t)part * S, (size_t)part * n * S, S, d);
            b.target1 = (uint64_t)(n - 1) * b.P * J;
          } else {
            for (int d = 0; d < n; ++d)
              if (d != me) add_push(T.push1, (size_t)d * S, 0, S, d);
            for (int d = 0; d < n; ++d)
              if (d != me) add_push(T.push2, 0, 0, S, d);
            b.target1 = (n - 1) * J;
            b.target2 = (n - 1) * J;
          }
          break;
        default:   // Gather/Broadcast
          if (!p2) {
            // process 1: to the root, then the root forwards all n payloads to
            // everyone (a rank's own payload is read locally, never sent back)
            if (!root) add_push(T.push1, 0, 0, S, 0);
            if (root)
              for (int d = 1; d < n; ++d)
                for (int r = 0; r < n; ++r) {
                  if (r == d) continue;
                  const size_t src0 = r == 0 ? b.send_off : b.dst1_off + (size_t)r * S;
                  add_push(T.push2, src0, (size_t)r * S, S, d);
                  add_push(T.push2_odd, r == 0 ? src0 : src0 + b.dst1_par, (size_t)r * S, S, d);
                }
            b.push2_arena = true;
            b.target1 = (n - 1) * J;
            b.target2 = root ? 0 : (n - 1) * J;
            break;
          }
          // process 2: to the root, then the root's a7 to all
          if (!root) add_push(T.push1, 0, 0, S, 0);
          if (root)
            for (int d = 1; d < n; ++d) add_push(T.push2, 0, 0, S, d);
          b.target1 = (n - 1) * J;
          b.target2 = root ? 0 : J;
          break;
      }
    }
  } else
  switch (b.routine) {
    case ESP_ALLGATHER:
      bufs(b.recv1, n * S);
      break;
    case ESP_ALLTOALL_ALLGATHER:
      bufs(b.recv1, n * S);
      if (!p2) bufs(b.recv2, (size_t)n * n * S);
      else { bufs(b.mid, S); bufs(b.recv2, n * S); }
      break;
    case ESP_GATHER_BROADCAST:
      bufs(b.recv1, n * S);
      if (p2) bufs(b.mid, S);
      break;
    default:   // ALLREDUCE (randomk / none), RS/AG, Reduce/Broadcast
      if (!w->sim) bufs(b.recv1, S);
      break;
  }

}

static void build_bucket(Layout& L, Bucket& b, HostTables& T, size_t zero_off_st, size_t& st_cursor,
                         size_t& hist_cursor, uint32_t* bflag) {
  Plan& p = L.p;
  esp_world_s* w = p.w;
  const int n = w->nranks, nl = w->nlocal;
  const bool none = b.kind == ESP_NONE;
  const bool sparse = is_sparse(b.kind);
  const bool dgc = b.kind == ESP_DGC || b.kind == ESP_TOPK;
  const bool quant = is_quant(b.kind);
  const float divisor = b.reduce == ESP_MEAN ? (float)n : 1.0f;
  const int nslots = (int)p.ctxs.size();
  const bool divis = b.routine == ESP_ALLTOALL_ALLGATHER || b.routine == ESP_GATHER_BROADCAST;
  const bool p2 = !none && divis && b.proc == 2;   // mid-scheme recompression (a7)
  b.p2 = p2;

  const size_t S = b.slot;
  auto bufs = [&](LocalBufs& lb, size_t per_rank) {
    size_t stride = round_up(per_rank, 256);
    size_t off = L.reserve(stride * nl);
    lb = LocalBufs{L.ptr<unsigned char>(off), stride};
    return off;
  };

  // ---- h1 segments
  const uint32_t h1_first = (uint32_t)T.h1.size();
  uint32_t unit_cursor = (uint32_t)T.h1_units.size();
  uint32_t group_cursor = (uint32_t)T.h1_groups.size();
  for (int lr = 0; lr < nl; ++lr) {
    for (size_t ti = 0; ti < b.tens.size(); ++ti) {
      esp_ctx_s* c = p.ctxs[b.tens[ti]];
      const int slot_idx = b.tens[ti];
      for (int part = 0; part < (none ? 1 : c->P); ++part) {
        const uint32_t lo = none ? 0 : c->plo[part], hi = none ? (uint32_t)c->N : c->phi[part];
        const uint32_t len = hi - lo;
        if (len == 0) continue;
        SegH1 s{};
        s.gptr = p.dyn_dev + slot_idx;
        s.goff = (uint64_t)lr * c->N + lo;
        s.step = p.dyn_dev + nslots + slot_idx;
        s.r = c->r ? c->r + (size_t)lr * c->N + lo : nullptr;
        s.chunk = b.send.base ? b.send.at(lr) + (size_t)part * S + b.coff[ti] : nullptr;
        s.lazy_in = c->lazy ? c->lazy + ((size_t)lr * c->P + part) * 2 : nullptr;
        s.lazy_out = const_cast<float*>(s.lazy_in);
        s.n = len;
        s.k = none ? 0 : c->pk[part];
        s.kpad = c->kpad;
        // compressors stream 4096-element tiles (stream_tma.cuh); NONE's pack uses kUnit
        const uint32_t nunits = div_up(len, none ? kUnit : kDgcTile);
        s.unit0 = unit_cursor;
        s.nunits = nunits;
        const uint32_t nruns = div_up(len, kRun);
        s.rpg = dgc ? dgc_rpg(len, s.k, c->cfg, b.rpg_cap) : kRunsPerGroup;
        s.ngroups = div_up(nruns, s.rpg);
        s.group0 = group_cursor;
        s.ef = c->cfg.error_feedback ? 1 : 0;
        s.unsampled = b.kind == ESP_TOPK ? 1 : 0;
        s.hash = b.kind == ESP_RANDOMK ? c->hash_base
                                       : host_splitmix64(c->tensor_id * 0x100000001b3ull + part);
        s.part = (uint32_t)part;
        s.rankterm = (b.kind == ESP_RANDOMK && !c->cfg.randomk_shared_indices) ? grank(w, lr) + 1 : 0;
        s.ratio = c->cfg.ratio;
        s.strata = dgc_strata(len, c->cfg.dgc_sample_rate);
        s.approx = c->cfg.dgc_approx ? 1 : 0;
        s.mom = c->u ? c->u + (size_t)lr * c->N + lo : nullptr;
        s.mcoef = (float)c->cfg.momentum;
        if (dgc && c->zrec) {
          s.zrec = c->zrec + (size_t)lr * c->zrec_stride + c->zrec_part[part];
          s.zcap = c->zcap;
        }
        // per-segment state (zeroed every call)
        size_t st_off = zero_off_st + st_cursor * sizeof(SelState);
        ++st_cursor;
        s.st = L.ptr<SelState>(st_off);
        s.bflag = bflag;
        if (dgc) {
          s.cand = L.ptr<uint2>(L.reserve((size_t)nruns * kRun * sizeof(uint2)));
          s.runcnt = L.ptr<uint32_t>(L.reserve((size_t)nruns * 4));
          s.hrep = dgc_hrep(s.k, s.ngroups);
          const size_t hbytes = round_up((size_t)dgc_hist_words(s.hrep) * 4, 256);
          s.gcnt = L.commit ? reinterpret_cast<uint32_t*>(p.zero + hist_cursor + hbytes) : nullptr;
          s.hist = L.commit ? reinterpret_cast<uint32_t*>(p.zero + hist_cursor) : nullptr;
          hist_cursor += hbytes + round_up((size_t)s.ngroups * 8, 256);
        }
        if (quant) {
          // per-run partial sums, every slot rewritten each call (SignOp::run)
          s.partial = L.ptr<double>(L.reserve((size_t)nruns * 16));
          s.pcount = L.ptr<uint32_t>(L.reserve((size_t)nruns * 8));
        }
        if (none) s.chunk = b.send.base ? b.send.at(lr) + b.coff[ti] : nullptr;
        T.h1.push_back(s);
        unit_cursor += nunits;
        if (dgc) group_cursor += s.ngroups;
        fill_unit_table(T.h1_units, (uint32_t)(T.h1.size() - 1 - h1_first), nunits);
        if (dgc) fill_unit_table(T.h1_groups, (uint32_t)(T.h1.size() - 1 - h1_first), s.ngroups);
      }
    }
  }
  b.nh1 = (int)(T.h1.size() - h1_first);
  b.h1_max_len = 0;
  for (int i = 0; i < b.nh1; ++i) b.h1_max_len = std::max(b.h1_max_len, T.h1[h1_first + i].n);
  // (segments of <= 1024 elements: dgc_small_kernel, one 256-thread CTA each;
  // up to 4096 the on-chip kernel's one-CTA path is faster when it fits)
  b.small = dgc && b.h1_max_len <= (uint32_t)kSample;
  // one-kernel h1 when the bucket fits the chip's shared memory: the smallest
  // tiles-per-CTA that gives every segment's CTAs a resident slot (grid <= #SMs);
  // the approximate-count mode keeps the chain (its result depends on the sample)
  b.onchip = false;
  if (dgc && (!b.small || b.h1_max_len > 1024) && dgc_mid_enabled()) {
    bool ok = true;
    for (int i = 0; i < b.nh1; ++i) ok = ok && !T.h1[h1_first + i].approx;
    int sms = 0, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 0;
    // segments of up to 4 tiles stay in one CTA (no global barriers: their
    // passes are shorter than a barrier round trip), larger ones spread out
    uint32_t max_tiles = 1;
    for (int i = 0; i < b.nh1; ++i) max_tiles = std::max(max_tiles, T.h1[h1_first + i].nunits);
    for (uint32_t tpc = std::min<uint32_t>(max_tiles, 4); ok && tpc <= dgc_mid_tpc_max(); ++tpc) {
      uint64_t ctas = 0;
      for (int i = 0; i < b.nh1; ++i) ctas += div_up(T.h1[h1_first + i].nunits, tpc);
      if (ctas <= (uint64_t)sms) {
        b.small = false;
        b.onchip = true;
        b.onchip_tpc = tpc;
        b.onchip_grid = (int)ctas;
        break;
      }
    }
  }
  {
    // algorithmic bytes of the streaming h1 pass: read g, read r,
    // write r = 12 B/elem with EF (4 B/elem without); sign adds 1/8 B/elem of
    // bits; NONE's pack reads and writes 4 B/elem
    uint64_t elems = 0;
    for (int i = 0; i < b.nh1; ++i) elems += T.h1[h1_first + i].n;
    const bool ef = p.ctxs[b.tens[0]]->cfg.error_feedback != 0;
    if (none) b.h1_bytes = 8 * elems;
    else if (quant) b.h1_bytes = (ef ? 12 : 4) * elems + elems / 8;
    else if (b.momentum != 0.0) b.h1_bytes = 20 * elems;   // + read u, write u (R20)
    else b.h1_bytes = (ef ? 12 : 4) * elems;
  }
  // unit/group tables refer to segment indices local to the bucket; the
  // unit0/group0 fields are relative to the bucket's own unit table
  {
    uint32_t u0 = 0, g0 = 0;
    for (int i = 0; i < b.nh1; ++i) {
      SegH1& s = T.h1[h1_first + i];
      s.unit0 = u0;
      u0 += s.nunits;
      s.group0 = g0;
      if (dgc) g0 += s.ngroups;
    }
    b.nh1_units = (int)u0;
    b.nh1_groups = dgc ? (int)g0 : 0;
  }

  // ---- a7 segments (process 2, the owner's mid-scheme recompression)
  const uint32_t a7_first = (uint32_t)T.a7.size();
  const uint32_t a7h2_first = (uint32_t)T.a7h2.size();
  if (p2) {
    // sparse: a dense temporary per local rank holds the decode-mean of each
    // tensor's n chunks (16-byte aligned per tensor); its base is read through
    // a static device word, like a gradient through the dyn array
    size_t tmp_elems = 0;
    for (int t : b.tens) tmp_elems += round_up(b.routine == ESP_ALLTOALL_ALLGATHER ? partition_len(p.ctxs[t]->N, n)
                                                                                   : p.ctxs[t]->N, 4);
    if (!quant) {
      bufs(b.a7tmp, 4 * tmp_elems);
      b.a7ptr = L.ptr<uint64_t>(L.reserve(8 * (size_t)nl));
    }
    uint32_t u0 = 0, g0 = 0, hu0 = 0;
    for (int lr = 0; lr < nl; ++lr) {
      const int j = grank(w, lr);
      if (b.routine == ESP_GATHER_BROADCAST && j != 0) continue;
      size_t toff_elems = 0;
      for (size_t ti = 0; ti < b.tens.size(); ++ti) {
        esp_ctx_s* c = p.ctxs[b.tens[ti]];
        const int slot_idx = b.tens[ti];
        uint32_t lo, hi;
        if (b.routine == ESP_ALLTOALL_ALLGATHER) { lo = c->plo[j]; hi = c->phi[j]; }
        else { lo = 0; hi = (uint32_t)c->N; }
        const uint32_t len = hi - lo;
        const size_t my_off = toff_elems;
        toff_elems += round_up(b.routine == ESP_ALLTOALL_ALLGATHER ? partition_len(c->N, n) : c->N, 4);
        if (len == 0) continue;
        // the n received chunks of this partition (rank order)
        const uint32_t piece0 = (uint32_t)T.a7_pieces.size();
        for (int r = 0; r < n; ++r) {
          if (b.fused && r == w->rank) {
            // push mode: my own chunk is read where h1 wrote it (rewritten only by
            // the next call's h1, after this call's consumers in stream order)
            unsigned char* mine = b.send.at(lr) + (size_t)(b.routine == ESP_ALLTOALL_ALLGATHER ? r : 0) * S + b.coff[ti];
            T.a7_pieces.push_back(mine);
            T.a7_pieces_odd.push_back(mine);
            continue;
          }
          T.a7_pieces.push_back(b.recv1.base ? b.recv1.at(lr) + (size_t)r * S + b.coff[ti] : nullptr);
          T.a7_pieces_odd.push_back(b.recv1.base && b.fused ? b.recv1.at(lr) + b.dst1_par + (size_t)r * S + b.coff[ti]
                                                            : nullptr);
        }
        SegH1 s{};
        s.r = c->r2 ? c->r2 + (size_t)lr * c->r2_len : nullptr;
        if (c->zrec2) {   // DGC / TOPK process 2: r2's deferred zeroing
          s.zrec = c->zrec2 + (size_t)lr * c->zrec2_stride;
          s.zcap = c->zcap;
        }
        s.lazy_in = c->lazy2 ? c->lazy2 + (size_t)lr * 2 : nullptr;
        s.lazy_out = const_cast<float*>(s.lazy_in);
        s.chunk = b.fused ? (b.stage.base ? b.stage.at(lr) + b.coff[ti] : nullptr)
                          : (b.mid.base ? b.mid.at(lr) + b.coff[ti] : nullptr);
        s.n = len;
        s.kpad = c->kpad;
        s.nunits = div_up(len, kDgcTile);
        s.unit0 = u0;
        u0 += s.nunits;
        s.ef = c->cfg.error_feedback ? 1 : 0;
        s.bflag = bflag ? bflag + 2 : nullptr;   // the a7 launch's own fallback / barrier words
        s.st = L.ptr<SelState>(zero_off_st + st_cursor * sizeof(SelState));
        ++st_cursor;
        if (quant) {
          s.npieces = (uint32_t)n;
          s.piece0 = piece0;
          s.divisor = divisor;
          // per-run partial sums, every slot rewritten each call (SignOp::run)
          s.partial = L.ptr<double>(L.reserve((size_t)div_up(s.n, kRun) * 16));
          s.pcount = L.ptr<uint32_t>(L.reserve((size_t)div_up(s.n, kRun) * 8));
        } else {
          // (i) decode-mean of the n chunks into the temporary (an h2 segment)
          SegH2 d{};
          d.optr = b.a7ptr ? b.a7ptr + lr : nullptr;
          d.ooff = my_off;
          d.step = p.dyn_dev + nslots + slot_idx;
          d.hash = c->hash_base;
          d.part = (uint32_t)(b.routine == ESP_ALLTOALL_ALLGATHER ? j : 0);
          d.n = len;
          d.k = k_of(len, c->cfg.ratio);
          d.kpad = c->kpad;
          d.npieces = (uint32_t)n;
          d.piece0 = piece0;
          d.divisor = divisor;
          d.nunits = div_up(len, dgc ? kTile : kUnit);
          d.unit0 = hu0;
          hu0 += d.nunits;
          for (int r = 0; r < n; ++r)
            T.a7h2_rankterms.push_back((b.kind == ESP_RANDOMK && !c->cfg.randomk_shared_indices) ? r + 1 : 0);
          if (dgc) {
            d.toff = L.ptr<uint32_t>(L.reserve((size_t)d.npieces * (d.nunits + 1) * 4));
            for (uint32_t r = 0; r < d.npieces; ++r)
              for (uint32_t e = 0; e < d.kpad; e += kOffJob)
                T.a7h2_off_jobs.push_back(make_uint4((uint32_t)(T.a7h2.size() - a7h2_first), r, e, 0));
          }
          T.a7h2.push_back(d);
          fill_unit_table(T.a7h2_units, (uint32_t)(T.a7h2.size() - 1 - a7h2_first), d.nunits);
          // (ii) the compressor's h1 on the temporary with r = r2 (alpha = 1/n resp. 1)
          s.gptr = b.a7ptr ? b.a7ptr + lr : nullptr;
          s.goff = my_off;
          s.step = p.dyn_dev + nslots + slot_idx;
          s.k = k_of(len, c->cfg.ratio);
          const uint32_t nruns = div_up(len, kRun);
          s.rpg = dgc ? dgc_rpg(len, s.k, c->cfg, b.rpg_cap) : kRunsPerGroup;
          s.ngroups = div_up(nruns, s.rpg);
          s.group0 = g0;
          s.unsampled = b.kind == ESP_TOPK ? 1 : 0;
          s.part = d.part;
          s.hash = b.kind == ESP_RANDOMK ? c->hash_base
                                         : host_splitmix64(c->tensor_id * 0x100000001b3ull + 0x9e37u + d.part);
          s.rankterm = (b.kind == ESP_RANDOMK && !c->cfg.randomk_shared_indices) ? (uint32_t)j + 1 : 0;
          s.ratio = c->cfg.ratio;
          s.strata = dgc_strata(len, c->cfg.dgc_sample_rate);
          s.approx = c->cfg.dgc_approx ? 1 : 0;
          if (dgc) {
            s.cand = L.ptr<uint2>(L.reserve((size_t)nruns * kRun * sizeof(uint2)));
            s.runcnt = L.ptr<uint32_t>(L.reserve((size_t)nruns * 4));
            s.hrep = dgc_hrep(s.k, s.ngroups);
            const size_t hbytes = round_up((size_t)dgc_hist_words(s.hrep) * 4, 256);
            s.gcnt = L.commit ? reinterpret_cast<uint32_t*>(p.zero + hist_cursor + hbytes) : nullptr;
            s.hist = L.commit ? reinterpret_cast<uint32_t*>(p.zero + hist_cursor) : nullptr;
            hist_cursor += hbytes + round_up((size_t)s.ngroups * 8, 256);
            g0 += s.ngroups;
            fill_unit_table(T.a7_groups, (uint32_t)(T.a7.size() - a7_first), s.ngroups);
          }
        }
        T.a7.push_back(s);
        fill_unit_table(T.a7_units, (uint32_t)(T.a7.size() - 1 - a7_first), s.nunits);
      }
    }
    b.na7 = (int)(T.a7.size() - a7_first);
    b.a7_max_len = 0;
    for (int i = 0; i < b.na7; ++i) b.a7_max_len = std::max(b.a7_max_len, T.a7[a7_first + i].n);
    b.na7_units = (int)u0;
    b.na7_groups = (int)g0;
    b.na7h2 = (int)(T.a7h2.size() - a7h2_first);
    b.na7h2_units = (int)hu0;
    double e = 0.0, m = 0.0;
    for (int i = 0; i < b.na7h2; ++i) {
      e += (double)T.a7h2[a7h2_first + i].kpad * T.a7h2[a7h2_first + i].npieces;
      m += (double)T.a7h2[a7h2_first + i].n;
    }
    b.a7h2_dense = h2_sparse_dense(e, m);
  }

  // ---- h2 segments
  const uint32_t h2_first = (uint32_t)T.h2.size();
  uint32_t u0 = 0;
  const bool tiles = dgc;
  for (int lr = 0; lr < nl; ++lr) {
    for (size_t ti = 0; ti < b.tens.size(); ++ti) {
      esp_ctx_s* c = p.ctxs[b.tens[ti]];
      const int slot_idx = b.tens[ti];
      const int nparts_out = (b.routine == ESP_ALLTOALL_ALLGATHER) ? c->P : 1;
      for (int part = 0; part < nparts_out; ++part) {
        const uint32_t lo = nparts_out > 1 ? c->plo[part] : 0;
        const uint32_t hi = nparts_out > 1 ? c->phi[part] : (uint32_t)c->N;
        const uint32_t len = hi - lo;
        if (len == 0) continue;
        SegH2 s{};
        s.optr = p.dyn_dev + slot_idx;
        s.ooff = (uint64_t)lr * c->N + lo;
        s.step = p.dyn_dev + nslots + slot_idx;
        s.hash = c->hash_base;
        s.part = (uint32_t)part;
        s.n = len;
        s.k = none ? 0 : k_of(len, c->cfg.ratio);
        s.kpad = c->kpad;
        s.piece0 = (uint32_t)T.h2_pieces.size();
        // fused: the parity-1 copy of the buffer h2 reads follows the parity-0 copy
        const size_t par_stride = b.routine == ESP_ALLGATHER ? b.dst1_par
                                  : (b.routine == ESP_ALLTOALL_ALLGATHER && !p2) ? b.dst1_par
                                                                                 : b.dst2_par;
        // process 2: the piece of partition part is the owner's recompression
        // (Randomk: drawn with rank = owner when indices are not shared)
        const uint32_t rt2 = (b.kind == ESP_RANDOMK && !c->cfg.randomk_shared_indices)
                                 ? (uint32_t)(b.routine == ESP_ALLTOALL_ALLGATHER ? part : 0) + 1 : 0;
        auto add_piece = [&](unsigned char* base, size_t off, uint32_t rankterm) {
          T.h2_pieces.push_back(base ? base + off : nullptr);
          T.h2_pieces_odd.push_back(base && b.fused ? base + off + par_stride : nullptr);
          T.rankterms.push_back(rankterm);
        };
        // push mode: a piece this rank produced itself is read from its local
        // source (no self copy); same pointer for both parities
        auto local_piece = [&](unsigned char* ptr, uint32_t rankterm) {
          T.h2_pieces.push_back(ptr);
          T.h2_pieces_odd.push_back(ptr);
          T.rankterms.push_back(rankterm);
        };
        const int me = w->rank;
        const uint32_t rt_shared = 0;
        auto rt_of = [&](int r) -> uint32_t {
          return (b.kind == ESP_RANDOMK && !c->cfg.randomk_shared_indices) ? (uint32_t)r + 1 : rt_shared;
        };
        switch (b.routine) {
          case ESP_ALLGATHER:
          case ESP_GATHER_BROADCAST:
            if (b.routine == ESP_GATHER_BROADCAST && p2) {
              if (b.fused && me == 0) local_piece(b.stage.at(lr) + b.coff[ti], rt2);
              else add_piece(b.mid.base ? b.mid.at(lr) : nullptr, b.coff[ti], rt2);
              s.npieces = 1;
              s.divisor = 1.0f;
            } else {
              for (int r = 0; r < n; ++r) {
                if (b.fused && r == me) local_piece(b.send.at(lr) + b.coff[ti], rt_of(r));
                else add_piece(b.recv1.base ? b.recv1.at(lr) : nullptr, (size_t)r * S + b.coff[ti], rt_of(r));
              }
              s.npieces = (uint32_t)n;
              s.divisor = divisor;
            }
            break;
          case ESP_ALLTOALL_ALLGATHER:
            if (!p2) {
              for (int r = 0; r < n; ++r)
                if (b.fused && r == me) local_piece(b.send.at(lr) + (size_t)part * S + b.coff[ti], rt_of(r));
                else add_piece(b.recv2.base ? b.recv2.at(lr) : nullptr,
                          (size_t)part * n * S + (size_t)r * S + b.coff[ti], rt_of(r));
              s.npieces = (uint32_t)n;
              s.divisor = divisor;
            } else {
              if (b.fused && part == me) local_piece(b.stage.at(lr) + b.coff[ti], rt2);
              else add_piece(b.recv2.base ? b.recv2.at(lr) : nullptr, (size_t)part * S + b.coff[ti], rt2);
              s.npieces = 1;
              s.divisor = 1.0f;
            }
            break;
          default:   // ALLREDUCE / RS-AG / Reduce-Broadcast
            if (w->sim) {
              for (int r = 0; r < n; ++r)
                add_piece(b.send.base ? b.send.at(r) : nullptr, b.coff[ti], 0);
              s.npieces = (uint32_t)n;
            } else {
              add_piece(b.recv1.base ? b.recv1.at(0) : nullptr, b.coff[ti], 0);
              s.npieces = 1;
            }
            s.divisor = divisor;
            break;
        }
        s.nunits = div_up(len, tiles ? kTile : quant ? kSignUnit : kUnit);
        s.unit0 = u0;
        u0 += s.nunits;
        if (tiles) {
          s.toff = L.ptr<uint32_t>(L.reserve((size_t)s.npieces * (s.nunits + 1) * 4));
          for (uint32_t r = 0; r < s.npieces; ++r)
            for (uint32_t e = 0; e < s.kpad; e += kOffJob)
              T.off_jobs.push_back(make_uint4((uint32_t)(T.h2.size() - h2_first), r, e, 0));
        }
        T.h2.push_back(s);
        fill_unit_table(T.h2_units, (uint32_t)(T.h2.size() - 1 - h2_first), s.nunits);
      }
    }
  }
  b.nh2 = (int)(T.h2.size() - h2_first);
  b.h2_max_pieces = 0;
  double h2_entries = 0.0, h2_elems = 0.0;
  for (int i = 0; i < b.nh2; ++i) {
    const SegH2& x = T.h2[h2_first + i];
    b.h2_max_pieces = std::max(b.h2_max_pieces, (int)x.npieces);
    h2_entries += (double)x.kpad * x.npieces;
    h2_elems += (double)x.n;
  }
  // small buckets take the CTA-tile kernel at any density: one launch instead of
  // the offset pass + the warp-per-tile kernel (their latency is the cost there)
  b.h2_dense = h2_sparse_dense(h2_entries, h2_elems) || h2_elems <= (double)(1u << 22);
  b.nh2_units = (int)u0;

  // per critical rank op counts of the cost table
  b.h1_calls = none ? 0 : (p2 ? 2 : 1);
  switch (b.routine) {
    case ESP_ALLGATHER: b.h2_pieces_count = n; break;
    case ESP_ALLTOALL_ALLGATHER: b.h2_pieces_count = !p2 ? (uint64_t)n * n : 2ull * n; break;
    case ESP_GATHER_BROADCAST: b.h2_pieces_count = p2 ? n + 1 : n; break;
    default: b.h2_pieces_count = none ? 0 : 1; break;
  }
}

// The bucket's cap on the finalize group length: 128 runs unless that leaves
// fewer than 2048 groups (warps) over the whole bucket -- a small bucket
// (config 1's 2^20 elements) wants many short groups, whose dependent-load
// chains run side by side, rather than a few long ones.
static uint32_t dgc_rpg_cap(const Plan& p, const Bucket& b) {
  uint32_t cap = kRunsPerGroup;
  for (; cap > 8; cap /= 2) {
    uint64_t groups = 0;
    for (int t : b.tens) {
      const esp_ctx_s* c = p.ctxs[t];
      for (int part = 0; part < c->P; ++part) {
        const uint64_t len = c->phi[part] - c->plo[part];
        if (len) groups += div_up(div_up(len, kRun), dgc_rpg(len, c->pk[part], c->cfg, cap));
      }
    }
    if (groups * (uint64_t)p.w->nlocal >= 2048) break;
  }
  return cap;
}

static void layout_plan(Plan& p, bool commit, HostTables& T) {
  Layout L{p, commit};
  for (auto& b : p.buckets)
    if (b.kind == ESP_DGC || b.kind == ESP_TOPK) b.rpg_cap = dgc_rpg_cap(p, b);
  p.arena.used = 0;
  const int nslots = (int)p.ctxs.size();
  size_t dyn_off = L.reserve(sizeof(uint64_t) * 2 * nslots);
  p.dyn_dev = L.ptr<uint64_t>(dyn_off);
  std::vector<HostTables> TBs(p.buckets.size());
  for (size_t i = 0; i < p.buckets.size(); ++i) layout_buffers(L, p.buckets[i], TBs[i]);
  // count segments to size the zero region: SelState per h1/a7 segment + hist per DGC segment
  size_t nst = 0, nhist = 0;
  for (auto& b : p.buckets) {
    const bool dgc = b.kind == ESP_DGC || b.kind == ESP_TOPK;
    for (int t : b.tens) {
      esp_ctx_s* c = p.ctxs[t];
      int segs = 0;
      for (int part = 0; part < (b.kind == ESP_NONE ? 1 : c->P); ++part) {
        const uint64_t len = b.kind == ESP_NONE ? c->N : c->phi[part] - c->plo[part];
        if (!len) continue;
        ++segs;
        // DGC: histograms + look-back status (one u64 per group of runs)
        if (dgc) {
          const uint32_t ng = (uint32_t)div_up(div_up(len, kRun), dgc_rpg(len, c->pk[part], c->cfg, b.rpg_cap));
          nhist += (round_up((size_t)dgc_hist_words(dgc_hrep(c->pk[part], ng)) * 4, 256) +
                    round_up((size_t)ng * 8, 256)) * p.w->nlocal;
        }
      }
      nst += (size_t)segs * p.w->nlocal;
      if (mid_scheme(c->cfg, c->routine)) {
        nst += (size_t)p.w->nlocal;   // a7 (upper bound)
        if (dgc)
          for (int lr = 0; lr < p.w->nlocal; ++lr) {
            // the owner's recompression of its partition (A2A) / the whole tensor (root)
            const int j = grank(p.w, lr);
            const uint64_t len = c->routine == ESP_ALLTOALL_ALLGATHER ? c->phi[j] - c->plo[j] : (j == 0 ? c->N : 0);
            if (!len) continue;
            const uint32_t ng =
                (uint32_t)div_up(div_up(len, kRun), dgc_rpg(len, k_of(len, c->cfg.ratio), c->cfg, b.rpg_cap));
            nhist += round_up((size_t)dgc_hist_words(dgc_hrep(k_of(len, c->cfg.ratio), ng)) * 4, 256) +
                     round_up((size_t)ng * 8, 256);
          }
      }
    }
  }
  const size_t st_bytes = round_up(nst * sizeof(SelState), 256);
  // per bucket: fallback flag + grid barrier of h1, the same two of a7
  const size_t flags_bytes = round_up(p.buckets.size() * 16, 256);
  p.zero_bytes = flags_bytes + st_bytes + nhist;
  size_t zero_off = L.reserve(p.zero_bytes);
  p.zero = commit ? p.arena.base + zero_off : nullptr;
  size_t st_cursor = 0, hist_cursor = flags_bytes + st_bytes;
  T = HostTables{};
  for (auto& b : p.buckets) {
    HostTables& TB = TBs[&b - p.buckets.data()];
    build_bucket(L, b, TB, zero_off + flags_bytes, st_cursor, hist_cursor,
                 commit ? reinterpret_cast<uint32_t*>(p.zero) + 4 * (&b - p.buckets.data()) : nullptr);
    // per-bucket device copies of the tables
    auto up = [&](const auto& vec, auto*& dst) {
      using E = typename std::decay<decltype(vec)>::type::value_type;
      size_t off = L.reserve(std::max<size_t>(1, vec.size()) * sizeof(E));
      dst = commit ? reinterpret_cast<typename std::decay<decltype(dst)>::type>(p.arena.base + off) : nullptr;
      if (commit && !vec.empty())
        ESP_CUDA(cudaMemcpy((void*)dst, vec.data(), vec.size() * sizeof(E), cudaMemcpyHostToDevice));
    };
    up(TB.h1, b.h1);
    up(TB.h1_units, b.h1_units);
    up(TB.h1_groups, b.h1_groups);
    up(TB.a7, b.a7);
    up(TB.a7_units, b.a7_units);
    up(TB.a7_groups, b.a7_groups);
    up(TB.a7h2, b.a7h2);
    up(TB.a7h2_units, b.a7h2_units);
    up(TB.a7h2_rankterms, b.a7h2_rankterms);
    up(TB.a7h2_off_jobs, b.a7h2_off_jobs);
    b.na7h2_off_jobs = (int)TB.a7h2_off_jobs.size();
    if (commit && b.a7ptr) {
      std::vector<uint64_t> bases(p.w->nlocal);
      for (int lr = 0; lr < p.w->nlocal; ++lr) bases[lr] = (uint64_t)(uintptr_t)b.a7tmp.at(lr);
      ESP_CUDA(cudaMemcpy(b.a7ptr, bases.data(), 8 * bases.size(), cudaMemcpyHostToDevice));
    }
    up(TB.a7_pieces, b.a7_pieces);
    if (b.fused) up(TB.a7_pieces_odd, b.a7_pieces_odd);
    up(TB.h2, b.h2);
    up(TB.h2_units, b.h2_units);
    up(TB.h2_pieces, b.h2_pieces);
    if (b.fused) up(TB.h2_pieces_odd, b.h2_pieces_odd);
    up(TB.rankterms, b.h2_rankterms);
    up(TB.off_jobs, b.h2_off_jobs);
    up(TB.push1, b.push1);
    up(TB.push2, b.push2);
    up(TB.push2_odd, b.push2_odd);
    up(TB.push1_mc, b.push1_mc);
    b.npush1_mc = (int)TB.push1_mc.size();
    b.npiece_ptrs = (int)TB.h2_pieces.size();
    b.npush1 = (int)TB.push1.size();
    b.npush2 = (int)TB.push2.size();
    b.push1_bytes = b.push2_bytes = b.push2_odd_bytes = 0;
    for (const PushJob& j : TB.push1) b.push1_bytes += j.bytes;
    for (const PushJob& j : TB.push2) b.push2_bytes += j.bytes;
    for (const PushJob& j : TB.push2_odd) b.push2_odd_bytes += j.bytes;
    b.nh2_off_jobs = (int)TB.off_jobs.size();
    if (commit) {
      // pad patterns of every chunk that kernels never touch (R: payload layout)
      // DGC / TOPK chunks carry the pad pattern (idx 0xFFFFFFFF, val +0) past
      // entry k: writers only store [0, k)
      auto pad_slots = [&](const LocalBufs& lb, int lr, size_t nslots_) {
        if (!lb.base) return;
        for (size_t q = 0; q < nslots_; ++q)
          for (size_t ti = 0; ti < b.tens.size(); ++ti) {
            esp_ctx_s* c = p.ctxs[b.tens[ti]];
            unsigned char* ch = lb.at(lr) + q * b.slot + b.coff[ti];
            ESP_CUDA(cudaMemset(ch, 0xFF, 4ull * c->kpad));
            ESP_CUDA(cudaMemset(ch + 4ull * c->kpad, 0, 4ull * c->kpad));
          }
      };
      const bool dgc_kind = b.kind == ESP_DGC || b.kind == ESP_TOPK;
      for (int lr = 0; lr < p.w->nlocal; ++lr) {
        if (dgc_kind) {
          pad_slots(b.send, lr, b.P);
          if (b.p2) {
            pad_slots(b.mid, lr, b.fused ? 2 : 1);   // fused: the G/B broadcast target (two parities)
            pad_slots(b.stage, lr, 1);
          }
        } else {
          ESP_CUDA(cudaMemset(b.send.at(lr), 0, b.P * b.slot));
          if (b.mid.base) ESP_CUDA(cudaMemset(b.mid.at(lr), 0, b.slot));
        }
        if (b.fused) {
          const int n = p.w->nranks;
          if (dgc_kind) {
            // every slot of both parity copies of every receive buffer
            const bool a2a1 = b.routine == ESP_ALLTOALL_ALLGATHER && !b.p2;
            pad_slots(b.recv1, lr, 2 * (size_t)n);
            pad_slots(b.recv2, lr, 2 * (size_t)n * (a2a1 ? n : 1));
          } else {
            if (b.recv1.base) ESP_CUDA(cudaMemset(b.recv1.at(lr), 0, 2ull * n * b.slot));
            if (b.recv2.base) ESP_CUDA(cudaMemset(b.recv2.at(lr), 0, 2ull * n * b.slot));
            if (b.mid.base) ESP_CUDA(cudaMemset(b.mid.at(lr), 0, 2ull * b.slot));
            if (b.stage.base) ESP_CUDA(cudaMemset(b.stage.at(lr), 0, b.slot));
          }
          ESP_CUDA(cudaMemset(p.arena.base + b.cnt_off, 0, 256));
        }
      }
    }
  }
}

// Fused buckets need every rank's arena mapped: exchange CUDA IPC handles of
// the arena through the NCCL communicator (a collective: done on the first
// esp_sync / esp_sync_many of the plan, which every rank calls) and build the
// destination / counter tables.
static void build_peer_tables(Plan& p, const std::vector<unsigned char*>& base);

// NVLS multicast for the plan's fused Allgather buckets (mcast.cu), decided
// collectively: every rank must support it and the world's mode must ask for
// it (auto: n >= 3, where one multicast store beats n - 1 unicast copies out
// of the sender's links; measured slower than one unicast copy at n = 2).
// The buckets' receive buffers and arrival counters move into the region
// (identical layout on every rank); h2's piece pointers are re-pointed there.
static void open_multicast(Plan& p, cudaStream_t st) {
  esp_world_s* w = p.w;
  const int n = w->nranks;
  const bool want = w->mc_mode == 1 || (w->mc_mode < 0 && n >= 3);
  bool any = false;
  for (const Bucket& b : p.buckets) any |= b.fused && b.routine == ESP_ALLGATHER;
  if (!want || !any || w->loopback) return;
  // every rank's verdict and rank 0's rendezvous token
  struct Info { uint64_t token; int32_t ok; int32_t pad; };
  Info mine{0, multicast_supported(w->dev) ? 1 : 0, 0};
  if (w->rank == 0) mine.token = host_splitmix64((uint64_t)getpid() * 0x9E3779B97F4A7C15ull ^ (uint64_t)(uintptr_t)&p);
  Info* d = nullptr;
  ESP_CUDA(cudaMalloc(&d, sizeof(Info) * (n + 1)));
  ESP_CUDA(cudaMemcpy(d + n, &mine, sizeof(Info), cudaMemcpyHostToDevice));
  ESP_NCCL(ncclAllGather(d + n, d, sizeof(Info), ncclUint8, w->comm, st));
  std::vector<Info> all(n);
  ESP_CUDA(cudaStreamSynchronize(st));
  ESP_CUDA(cudaMemcpy(all.data(), d, sizeof(Info) * n, cudaMemcpyDeviceToHost));
  cudaFree(d);
  for (const Info& i : all)
    if (!i.ok) return;   // one rank without multicast: unicast pushes everywhere
  // region layout: per Allgather bucket [2 parities][n slots][S] then 4 counters
  std::vector<size_t> off(p.buckets.size(), 0);
  size_t cursor = 0;
  for (size_t i = 0; i < p.buckets.size(); ++i) {
    const Bucket& b = p.buckets[i];
    if (!(b.fused && b.routine == ESP_ALLGATHER)) continue;
    off[i] = round_up(cursor, 256);
    cursor = off[i] + round_up(2ull * n * b.slot, 256) + 256;
  }
  p.mcr.reset(mcast_create(w, cursor, all[0].token, w->mc_seq++, st));
  unsigned char* uc = reinterpret_cast<unsigned char*>(p.mcr->uc_va);
  unsigned char* mcv = reinterpret_cast<unsigned char*>(p.mcr->mc_va);
  for (size_t i = 0; i < p.buckets.size(); ++i) {
    Bucket& b = p.buckets[i];
    if (!(b.fused && b.routine == ESP_ALLGATHER)) continue;
    const size_t recv_bytes = 2ull * n * b.slot;
    const size_t cnt_off = off[i] + round_up(recv_bytes, 256);
    // h2 reads the pieces from this rank's copy of the region
    auto repoint = [&](const unsigned char** dev_arr) {
      if (!dev_arr || b.npiece_ptrs == 0) return;
      std::vector<const unsigned char*> h(b.npiece_ptrs);
      ESP_CUDA(cudaMemcpy(h.data(), dev_arr, sizeof(void*) * h.size(), cudaMemcpyDeviceToHost));
      for (auto& q : h)
        if (q >= b.recv1.base && q < b.recv1.base + recv_bytes) q = uc + off[i] + (q - b.recv1.base);
      ESP_CUDA(cudaMemcpy(dev_arr, h.data(), sizeof(void*) * h.size(), cudaMemcpyHostToDevice));
    };
    repoint(b.h2_pieces);
    repoint(b.h2_pieces_odd);
    b.recv1.base = uc + off[i];
    b.my_cnt = reinterpret_cast<unsigned long long*>(uc + cnt_off);
    b.mc_recv = mcv + off[i];
    b.mc_cnt = reinterpret_cast<unsigned long long*>(mcv + cnt_off);
    b.target1 = (uint64_t)n * b.npush1_mc;   // every rank's jobs bump every counter, mine included
    b.mc = true;
  }
}

static void open_peers(Plan& p, cudaStream_t st) {
  esp_world_s* w = p.w;
  const int n = w->nranks;
  cudaIpcMemHandle_t mine;
  ESP_CUDA(cudaIpcGetMemHandle(&mine, p.arena.base));
  unsigned char* dbuf = nullptr;
  ESP_CUDA(cudaMalloc(&dbuf, sizeof(mine) * (n + 1)));
  ESP_CUDA(cudaMemcpy(dbuf + sizeof(mine) * n, &mine, sizeof(mine), cudaMemcpyHostToDevice));
  ESP_NCCL(ncclAllGather(dbuf + sizeof(mine) * n, dbuf, sizeof(mine), ncclUint8, w->comm, st));
  std::vector<cudaIpcMemHandle_t> all(n);
  ESP_CUDA(cudaStreamSynchronize(st));
  ESP_CUDA(cudaMemcpy(all.data(), dbuf, sizeof(mine) * n, cudaMemcpyDeviceToHost));
  cudaFree(dbuf);
  std::vector<unsigned char*> base(n);
  p.peer_bases.assign(n, nullptr);
  for (int q = 0; q < n; ++q) {
    if (q == w->rank) {
      base[q] = p.arena.base;
    } else {
      void* ptr = nullptr;
      ESP_CUDA(cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess));
      p.peer_bases[q] = ptr;
      base[q] = static_cast<unsigned char*>(ptr);
    }
  }
  build_peer_tables(p, base);
  open_multicast(p, st);
}

// destination / counter tables of every fused bucket from the n arena bases
static void build_peer_tables(Plan& p, const std::vector<unsigned char*>& base) {
  esp_world_s* w = p.w;
  const int n = w->nranks;
  auto upload = [](auto& dev, const auto& host) {
    ESP_CUDA(cudaMalloc(&dev, sizeof(host[0]) * host.size()));
    ESP_CUDA(cudaMemcpy(dev, host.data(), sizeof(host[0]) * host.size(), cudaMemcpyHostToDevice));
  };
  for (auto& b : p.buckets) {
    if (!b.fused) continue;
    // my slot in every rank q's phase-1/2 buffer and q's arrival counters,
    // per call parity ([parity][q])
    std::vector<unsigned char*> dsts(2 * n), dsts2(2 * n);
    std::vector<unsigned long long*> cnts(2 * n), cnts2(2 * n);
    for (int par = 0; par < 2; ++par)
      for (int q = 0; q < n; ++q) {
        dsts[par * n + q] = base[q] + b.dst1_off + par * b.dst1_par + (size_t)w->rank * b.dst1_slot;
        dsts2[par * n + q] = base[q] + b.dst2_off + par * b.dst2_par + (size_t)w->rank * b.dst2_slot;
        unsigned long long* c = reinterpret_cast<unsigned long long*>(base[q] + b.cnt_off);
        cnts[par * n + q] = c + par;
        cnts2[par * n + q] = c + 2 + par;
      }
    b.my_cnt = reinterpret_cast<unsigned long long*>(p.arena.base + b.cnt_off);
    upload(b.dsts, dsts);
    upload(b.dsts2, dsts2);
    upload(b.cnts, cnts);
    upload(b.cnts2, cnts2);
  }
  p.peers_ready = true;
}

// Plans are cached per world in LRU order (most recent last) and bounded by
// w->plan_cap.  Evicting a fused plan is safe without a cross-rank barrier:
// its last call has completed here (the eviction synchronizes), so every
// peer's pushes into this arena have landed (they precede our wait kernel's
// arrivals), and ranks run the same call sequence, so no peer calls it again.
void trim_plans(esp_world_s* w) {
  if (w->plans.size() <= w->plan_cap) return;
  cudaDeviceSynchronize();
  while (w->plans.size() > w->plan_cap) {
    delete w->plans.front();
    w->plans.erase(w->plans.begin());
  }
}

Plan* find_plan(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs) {
  for (size_t i = w->plans.size(); i-- > 0;)   // most recently used first
    if (w->plans[i]->ctxs == ctxs) {
      Plan* up = w->plans[i];
      if (i + 1 != w->plans.size()) {
        w->plans.erase(w->plans.begin() + i);
        w->plans.push_back(up);
      }
      return up;
    }
  return nullptr;
}

Plan* get_plan(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs) {
  if (Plan* up = find_plan(w, ctxs)) return up;
  auto p = std::make_unique<Plan>();
  p->w = w;
  p->ctxs = ctxs;
  // ---- bucketing: group by (kind, routine, reduce, process) in order of first
  // appearance, split each class at bucket_elems elements per rank
  const uint64_t cap = w->bucket_elems ? w->bucket_elems : (512ull << 20);
  std::vector<std::pair<std::tuple<int, int, int, int, double, int>, std::vector<int>>> classes;
  for (int i = 0; i < (int)ctxs.size(); ++i) {
    auto key = std::make_tuple(ctxs[i]->cfg.kind, ctxs[i]->routine, ctxs[i]->cfg.reduce, process_of(ctxs[i]->cfg),
                               ctxs[i]->cfg.momentum, ctxs[i]->cfg.error_feedback);
    auto it = std::find_if(classes.begin(), classes.end(), [&](auto& c) { return c.first == key; });
    if (it == classes.end()) classes.push_back({key, {i}});
    else it->second.push_back(i);
  }
  for (auto& cl : classes) {
    Bucket b;
    b.kind = std::get<0>(cl.first);
    b.routine = std::get<1>(cl.first);
    b.reduce = std::get<2>(cl.first);
    b.proc = std::get<3>(cl.first);
    b.momentum = std::get<4>(cl.first);
    b.ef = std::get<5>(cl.first) != 0;
    uint64_t elems = 0;
    for (int i : cl.second) {
      if (!b.tens.empty() && elems + ctxs[i]->N > cap) {
        p->buckets.push_back(b);
        b.tens.clear();
        elems = 0;
      }
      b.tens.push_back(i);
      elems += ctxs[i]->N;
    }
    if (!b.tens.empty()) p->buckets.push_back(b);
  }
  HostTables T;
  layout_plan(*p, false, T);
  p->arena.alloc();
  layout_plan(*p, true, T);
  for (auto& b : p->buckets) {
    ESP_CUDA(cudaEventCreateWithFlags(&b.ev_h1, cudaEventDisableTiming));
    ESP_CUDA(cudaEventCreateWithFlags(&b.ev_comm, cudaEventDisableTiming));
    ESP_CUDA(cudaEventCreateWithFlags(&b.ev_stream, cudaEventDisableTiming));
  }
  ESP_CUDA(cudaMallocHost(&p->dyn_host,
                          sizeof(uint64_t) * 2 * std::max<size_t>(1, ctxs.size()) * Plan::kDynSlots));
  for (auto& e : p->dyn_ev) ESP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& b : p->buckets)
    if (b.kind == ESP_RANDOMK) p->needs_step = true;
  w->plans.push_back(p.release());
  Plan* mine = w->plans.back();
  trim_plans(w);
  return mine;
}

void drop_plans_with(esp_world_s* w, esp_ctx_s* c) {
  auto& v = w->plans;
  for (auto it = v.begin(); it != v.end();) {
    if (std::find((*it)->ctxs.begin(), (*it)->ctxs.end(), c) != (*it)->ctxs.end()) {
      cudaStreamSynchronize(w->comm_stream);
      cudaDeviceSynchronize();
      delete *it;
      it = v.erase(it);
    } else {
      ++it;
    }
  }
}

void clear_plans(esp_world_s* w) {
  if (!w->plans.empty()) cudaDeviceSynchronize();
  for (Plan* p : w->plans) delete p;
  w->plans.clear();
}

// ------------------------------------------------------------------ execution
static void upload_dyn(Plan& p, const float* const* grads, cudaStream_t st) {
  const size_t ns = p.ctxs.size();
  // nothing any kernel reads changed (same gradient buffers, no step-keyed
  // kernel): the device copy from the previous call is still exact
  if (!p.needs_step && p.dyn_last.size() == ns && std::equal(p.dyn_last.begin(), p.dyn_last.end(), grads))
    return;
  const int slot = p.dyn_slot;
  p.dyn_slot = (slot + 1) % Plan::kDynSlots;
  if (p.dyn_pending[slot]) ESP_CUDA(cudaEventSynchronize(p.dyn_ev[slot]));
  uint64_t* h = p.dyn_host + (size_t)slot * 2 * ns;
  for (size_t i = 0; i < ns; ++i) {
    h[i] = (uint64_t)(uintptr_t)grads[i];
    h[ns + i] = p.ctxs[i]->step;
  }
  ESP_CUDA(cudaMemcpyAsync(p.dyn_dev, h, sizeof(uint64_t) * 2 * ns, cudaMemcpyHostToDevice, st));
  ESP_CUDA(cudaEventRecord(p.dyn_ev[slot], st));
  p.dyn_pending[slot] = true;
  p.dyn_last.assign(grads, grads + ns);
}

static void probe_pair(esp_world_s* w, cudaEvent_t* e0, cudaEvent_t* e1, uint64_t bytes) {
  while (w->probe_pool.size() < 2 * (w->probe_used + 1)) {
    cudaEvent_t e;
    ESP_CUDA(cudaEventCreate(&e));
    w->probe_pool.push_back(e);
  }
  *e0 = w->probe_pool[2 * w->probe_used];
  *e1 = w->probe_pool[2 * w->probe_used + 1];
  w->probe_bytes.resize(w->probe_used + 1);
  w->probe_bytes[w->probe_used] = bytes;
  ++w->probe_used;
}

// h1 of a bucket: the payload is written locally (send); in a fused bucket
// push_kernel then moves it to the peers (run_comm).  `fin` (DGC, several
// buckets): the finalize chain (latency-bound: radix select and ordered write
// over the candidates) runs there after the streaming pass, so that it
// overlaps the next bucket's HBM-bound streaming pass on `st` (a9).
// Returns the stream on which the bucket's payload is complete.
static cudaStream_t run_h1(Plan& p, Bucket& b, cudaStream_t st, cudaStream_t fin = nullptr) {
  cudaStream_t done = st;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p.w->probe && b.nh1_units) probe_pair(p.w, &e0, &e1, b.h1_bytes);
  const bool dgc = b.kind == ESP_DGC || b.kind == ESP_TOPK;
  const bool sign = b.kind == ESP_EFSIGNSGD || b.kind == ESP_ONEBIT;
  if (e0 && !dgc && !sign) ESP_CUDA(cudaEventRecord(e0, st));
  switch (b.kind) {
    case ESP_DGC: case ESP_TOPK:
      if (b.small) {   // every segment fits one CTA: the whole h1 in one kernel
        if (e0) ESP_CUDA(cudaEventRecord(e0, st));
        launch_dgc_small(b.h1, b.nh1, st);
        if (e1) ESP_CUDA(cudaEventRecord(e1, st));
      } else if (b.onchip) {   // the bucket fits on chip: the whole h1 in one kernel
        if (e0) ESP_CUDA(cudaEventRecord(e0, st));
        launch_dgc_mid(b.h1, b.nh1, b.onchip_tpc, b.onchip_grid, st);
        if (e1) ESP_CUDA(cudaEventRecord(e1, st));
      } else if (fin) {
        launch_dgc_stream(b.h1, b.nh1, b.h1_units, b.nh1_units, st, e0, e1, b.momentum != 0.0);
        ESP_CUDA(cudaEventRecord(b.ev_stream, st));
        ESP_CUDA(cudaStreamWaitEvent(fin, b.ev_stream, 0));
        launch_dgc_finalize(b.h1, b.nh1, b.h1_groups, b.nh1_groups, fin);
        done = fin;
      } else {
        launch_dgc_h1(b.h1, b.nh1, b.h1_units, b.nh1_units, b.h1_groups, b.nh1_groups, st, e0, e1,
                      b.momentum != 0.0);
      }
      break;
    case ESP_RANDOMK: launch_randomk_h1(b.h1, b.h1_units, b.nh1_units, st); break;
    case ESP_EFSIGNSGD:
    case ESP_ONEBIT: {
      const int k = b.kind == ESP_EFSIGNSGD ? K_EFSIGN : K_ONEBIT;
      launch_sign_h1_tma(k, b.h1, b.nh1, b.h1_units, b.nh1_units, nullptr, st, b.h1_max_len, e0, e1);
      break;
    }
    default: launch_pack(b.h1, b.h1_units, b.nh1_units, st); break;
  }
  if (e1 && !dgc && !sign) ESP_CUDA(cudaEventRecord(e1, st));
  ESP_CUDA(cudaGetLastError());
  for (int lr = 0; lr < p.w->nlocal; ++lr) p.w->counters[lr].h1_calls += b.h1_calls * b.tens.size();
  return done;
}

// ESP_DEBUG_SYNC=1: synchronize after each phase of the collective layer and
// name the one that failed (debugging aid; off by default)
static void dbg(const char* what, cudaStream_t st) {
  static const bool on = [] {
    const char* e = getenv("ESP_DEBUG_SYNC");
    return e && atoi(e) != 0;
  }();
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(st);
  fprintf(stderr, "[esp] %s: %s\n", what, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  fflush(stderr);
}

static void run_mid(Plan& p, Bucket& b, cudaStream_t cs) {
  const int k = b.kind == ESP_EFSIGNSGD ? K_EFSIGN : K_ONEBIT;
  const unsigned char* const* pieces = (b.fused && (b.epoch & 1)) ? b.a7_pieces_odd : b.a7_pieces;
  if (!is_quant(b.kind)) {
    // sparse process 2: decode-mean of the n chunks into the temporary, then the
    // compressor's h1 on it (r = r2), output to stage (push) or mid
    if (b.kind == ESP_RANDOMK) {
      launch_h2_randomk(b.a7h2, b.a7h2_units, b.na7h2_units, pieces, b.a7h2_rankterms, cs);
      dbg("a7 decode (randomk)", cs);
      launch_randomk_h1(b.a7, b.a7_units, b.na7_units, cs);
    } else {
      launch_h2_sparse(b.a7h2, b.a7h2_units, b.na7h2_units, b.a7h2_off_jobs, b.na7h2_off_jobs, pieces,
                       p.w->nranks, b.a7h2_dense, cs);
      dbg("a7 decode (sparse)", cs);
      launch_dgc_h1(b.a7, b.na7, b.a7_units, b.na7_units, b.a7_groups, b.na7_groups, cs);
    }
    dbg("a7 recompress", cs);
  } else {
    launch_sign_h1_tma(k, b.a7, b.na7, b.a7_units, b.na7_units, pieces, cs, b.a7_max_len, nullptr, nullptr,
                       p.w->nranks);
  }
  ESP_CUDA(cudaGetLastError());
}

// Fused collective of a bucket in three stages.  Every rank runs them in
// order; across ranks, stage s of any rank may depend only on stages < s of
// the others (stage 1 pushes the first payloads, stage 2 waits for them and
// runs the owner's / root's a7 and second push, stage 3 waits for those), so
// the loopback executor can run all ranks' stage 1, then all stage 2, then all
// stage 3, on one stream with every wait already satisfied when it starts.
// push_kernel moves the local payloads (h1's send, then a7's stage) to the
// peers; a wait kernel blocks on the counter of this call's parity (monotonic
// across that parity's calls).  The byte counters record the routine's
// logical traffic (the cost table).
static void fused_stage(Plan& p, Bucket& b, int stage, cudaStream_t cs, cudaEvent_t mid0, cudaEvent_t mid1) {
  esp_world_s* w = p.w;
  const int n = w->nranks;
  const size_t S = b.slot;
  const bool quant = b.p2;   // a mid-scheme recompression between the two phases
  const int par = (int)(b.epoch & 1);
  const unsigned long long e1 = (b.epoch >> 1) + 1;   // calls of this parity so far, this one included
  unsigned long long* cnt1 = b.my_cnt + par;          // [2 * phase + parity]
  unsigned long long* cnt2 = b.my_cnt + 2 + par;
  const bool root = w->rank == 0;
  auto push2 = [&] {
    if (b.push2_arena)
      launch_push(par ? b.push2_odd : b.push2, b.npush2, p.arena.base, b.dsts2 + par * n, b.cnts2 + par * n, cs);
    else
      launch_push(b.push2, b.npush2, b.stage.at(0), b.dsts2 + par * n, b.cnts2 + par * n, cs);
    w->counters[0].pushed += par && b.push2_arena ? b.push2_odd_bytes : b.push2_bytes;
    dbg("push phase 2", cs);
  };
  auto mid = [&] {
    if (mid0) ESP_CUDA(cudaEventRecord(mid0, cs));
    run_mid(p, b, cs);
    if (mid1) ESP_CUDA(cudaEventRecord(mid1, cs));
  };
  auto wait = [&](unsigned long long* c, uint64_t target) {
    launch_wait_arrivals(c, e1 * target, w->wait_err, w->wait_timeout_ns, cs);
    dbg("wait", cs);
  };
  if (stage == 1) {
    if (b.mc) {   // one multicast store of my slot into every rank's receive buffer
      launch_push_mc(b.push1_mc, b.npush1_mc, b.send.at(0), b.mc_recv + (size_t)par * n * S + (size_t)w->rank * S,
                     b.mc_cnt + par, cs);
      w->counters[0].pushed += S;
    } else {
      launch_push(b.push1, b.npush1, b.send.at(0), b.dsts + par * n, b.cnts + par * n, cs);
      w->counters[0].pushed += b.push1_bytes;
    }
    dbg("push phase 1", cs);
    return;
  }
  switch (b.routine) {
    case ESP_ALLGATHER:
      if (stage == 2) {
        count_coll(w, 0, ESP_OP_ALLGATHER, (n - 1) * S, (n - 1) * S);
        wait(cnt1, b.target1);
      }
      break;
    case ESP_ALLTOALL_ALLGATHER:
      if (stage == 2) {
        count_coll(w, 0, ESP_OP_ALLTOALL, (n - 1) * S, (n - 1) * S);
        wait(cnt1, b.target1);
        if (quant) {
          mid();
          push2();
          count_coll(w, 0, ESP_OP_ALLGATHER, (n - 1) * S, (n - 1) * S);
        } else {
          count_coll(w, 0, ESP_OP_ALLGATHER, (n - 1) * n * S, (n - 1) * n * S);
        }
      } else if (quant) {
        wait(cnt2, b.target2);
      }
      break;
    default:   // Gather/Broadcast
      if (stage == 2) {
        count_coll(w, 0, ESP_OP_GATHER, root ? 0 : S, root ? (n - 1) * S : 0);
        if (root) {
          wait(cnt1, b.target1);
          if (quant) mid();   // process 2: the root's mid-scheme recompression
          push2();            // process 1: the root forwards the n payloads
        }
        const size_t bc = quant ? S : (size_t)n * S;
        count_coll(w, 0, ESP_OP_BROADCAST, root ? bc : 0, root ? 0 : bc);
      } else {
        wait(cnt2, b.target2);
      }
      break;
  }
  ESP_CUDA(cudaGetLastError());
}

static void run_comm(Plan& p, Bucket& b, cudaStream_t cs, cudaEvent_t mid0, cudaEvent_t mid1) {
  esp_world_s* w = p.w;
  const int n = w->nranks;
  const size_t S = b.slot;
  const bool quant = b.p2;   // a mid-scheme recompression between the two phases
  if (b.fused) {
    for (int stage = 1; stage <= 3; ++stage) fused_stage(p, b, stage, cs, mid0, mid1);
    return;
  }
  switch (b.routine) {
    case ESP_ALLGATHER:
      coll_allgather(w, b.send, b.recv1, S, cs);
      break;
    case ESP_ALLTOALL_ALLGATHER:
      coll_alltoall(w, b.send, b.recv1, S, cs);
      if (quant) {
        if (mid0) ESP_CUDA(cudaEventRecord(mid0, cs));
        run_mid(p, b, cs);
        if (mid1) ESP_CUDA(cudaEventRecord(mid1, cs));
        coll_allgather(w, b.mid, b.recv2, S, cs);
      } else {
        coll_allgather(w, b.recv1, b.recv2, (size_t)n * S, cs);
      }
      break;
    case ESP_GATHER_BROADCAST:
      coll_gather(w, b.send, b.recv1, S, cs);
      if (quant) {
        if (mid0) ESP_CUDA(cudaEventRecord(mid0, cs));
        run_mid(p, b, cs);
        if (mid1) ESP_CUDA(cudaEventRecord(mid1, cs));
        coll_broadcast(w, b.mid, S, cs);
      } else {
        coll_broadcast(w, b.recv1, (size_t)n * S, cs);
      }
      break;
    default: {
      // ALLREDUCE (NONE or shared-index Randomk values), RS/AG, Reduce/Broadcast
      const size_t count = b.kind == ESP_NONE ? b.none_count : S / 4;
      const uint64_t M = b.kind == ESP_NONE ? b.none_bytes : S;   // logical bytes
      for (int lr = 0; lr < w->nlocal; ++lr) {
        const bool root = (w->sim ? lr : w->rank) == 0;
        if (b.routine == ESP_ALLREDUCE) {
          count_coll(w, lr, ESP_OP_ALLREDUCE, 2ull * (n - 1) * M / n, 2ull * (n - 1) * M / n);
        } else if (b.routine == ESP_REDUCESCATTER_ALLGATHER) {
          count_coll(w, lr, ESP_OP_REDUCESCATTER, (n - 1) * M / n, (n - 1) * M / n);
          count_coll(w, lr, ESP_OP_ALLGATHER, (n - 1) * M / n, (n - 1) * M / n);
        } else {
          count_coll(w, lr, ESP_OP_REDUCE, root ? 0 : M, root ? (n - 1) * M : 0);
          count_coll(w, lr, ESP_OP_BROADCAST, root ? (n > 1 ? M : 0) : 0, root ? 0 : M);
        }
      }
      if (w->sim) {
        // executed by h2, which reads every virtual rank's packed buffer
      } else if (b.routine == ESP_ALLREDUCE) {
        coll_allreduce_f32(w, b.send, b.recv1, count, cs);
      } else if (b.routine == ESP_REDUCESCATTER_ALLGATHER) {
        LocalBufs shard{b.recv1.base + (size_t)w->rank * (count / n) * 4, b.recv1.stride};
        coll_reducescatter_f32(w, b.send, shard, count, cs);
        coll_allgather_inplace_f32(w, b.recv1, count / n, cs);
      } else {
        coll_reduce_f32(w, b.send, b.recv1, count, cs);
        if (n > 1) ESP_NCCL(ncclBroadcast(b.recv1.at(0), b.recv1.at(0), 4 * count, ncclUint8, 0, w->comm, cs));
      }
      break;
    }
  }
}

static void run_h2(Plan& p, Bucket& b, cudaStream_t st) {
  switch (b.kind) {
    case ESP_DGC: case ESP_TOPK:
      launch_h2_sparse(b.h2, b.h2_units, b.nh2_units, b.h2_off_jobs, b.nh2_off_jobs,
                       (b.fused && (b.epoch & 1)) ? b.h2_pieces_odd : b.h2_pieces, b.h2_max_pieces, b.h2_dense, st);
      break;
    case ESP_RANDOMK:
      launch_h2_randomk(b.h2, b.h2_units, b.nh2_units, (b.fused && (b.epoch & 1)) ? b.h2_pieces_odd : b.h2_pieces,
                        b.h2_rankterms, st);
      break;
    case ESP_EFSIGNSGD:
    case ESP_ONEBIT:
      launch_h2_sign(b.kind == ESP_EFSIGNSGD ? K_EFSIGN : K_ONEBIT, b.h2, b.h2_units, b.nh2_units,
                     (b.fused && (b.epoch & 1)) ? b.h2_pieces_odd : b.h2_pieces, b.h2_max_pieces, st);
      break;
    default: launch_h2_dense(b.h2, b.h2_units, b.nh2_units, b.h2_pieces, st); break;
  }
  ESP_CUDA(cudaGetLastError());
  for (int lr = 0; lr < p.w->nlocal; ++lr) p.w->counters[lr].h2_pieces += b.h2_pieces_count * b.tens.size();
}

static cudaEvent_t tev(esp_world_s* w, size_t i) {
  while (w->tev.size() <= i) {
    cudaEvent_t e;
    ESP_CUDA(cudaEventCreate(&e));
    w->tev.push_back(e);
  }
  return w->tev[i];
}

static bool graphs_enabled() {
  static const bool on = [] {
    const char* e = getenv("ESP_GRAPHS");   // ESP_GRAPHS=0: launch every kernel directly (debugging)
    return !(e && e[0] == '0');
  }();
  return on;
}

static int graph_key() {
  const char* ff = getenv("ESP_DGC_FORCE_FALLBACK");   // a test hook read at launch time
  return ff ? atoi(ff) : 0;
}

// run `body(stream)` as a graph: replay the cached one, or capture it on the
// world's capture stream (the caller's stream may be the legacy default
// stream, which cannot be captured) and launch it on `st`
template <class F>
static void run_graphed(Plan& p, GraphCache& g, cudaStream_t st, F body) {
  esp_world_s* w = p.w;
  const int key = graph_key();
  if (!g.exec || g.key != key) {
    if (g.exec) ESP_CUDA(cudaGraphExecDestroy(g.exec));
    g.exec = nullptr;
    const std::vector<esp_counters_t> before = w->counters;
    const uint64_t l0 = esp_launch_count();
    ESP_CUDA(cudaStreamBeginCapture(w->cap_stream, cudaStreamCaptureModeRelaxed));
    try {
      body(w->cap_stream);
    } catch (...) {
      cudaGraph_t gr = nullptr;
      cudaStreamEndCapture(w->cap_stream, &gr);
      if (gr) cudaGraphDestroy(gr);
      throw;
    }
    cudaGraph_t graph = nullptr;
    ESP_CUDA(cudaStreamEndCapture(w->cap_stream, &graph));
    const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    ESP_CUDA(e);
    g.key = key;
    g.launches = esp_launch_count() - l0;
    g.delta.assign(w->counters.size(), esp_counters_t{});
    for (size_t lr = 0; lr < w->counters.size(); ++lr) {
      const esp_counters_t &a = before[lr], &b = w->counters[lr];
      esp_counters_t& d = g.delta[lr];
      for (int o = 0; o < ESP_NUM_OPS; ++o) {
        d.calls[o] = b.calls[o] - a.calls[o];
        d.sent[o] = b.sent[o] - a.sent[o];
        d.recv[o] = b.recv[o] - a.recv[o];
      }
      d.h1_calls = b.h1_calls - a.h1_calls;
      d.h2_pieces = b.h2_pieces - a.h2_pieces;
      d.pushed = b.pushed - a.pushed;
    }
    ESP_CUDA(cudaGraphLaunch(g.exec, st));   // this call's work (the capture executed nothing)
    return;
  }
  ESP_CUDA(cudaGraphLaunch(g.exec, st));
  count_launches((int)g.launches);
  for (size_t lr = 0; lr < w->counters.size(); ++lr) {
    esp_counters_t& c = w->counters[lr];
    const esp_counters_t& d = g.delta[lr];
    for (int o = 0; o < ESP_NUM_OPS; ++o) {
      c.calls[o] += d.calls[o];
      c.sent[o] += d.sent[o];
      c.recv[o] += d.recv[o];
    }
    c.h1_calls += d.h1_calls;
    c.h2_pieces += d.h2_pieces;
    c.pushed += d.pushed;
  }
}

// a plan whose device work is identical on every call: no fused collective
// (call parities) and no NCCL call (sim worlds and single-rank worlds only)
static bool graphable(const Plan& p) {
  const esp_world_s* w = p.w;
  if (!graphs_enabled() || w->timing || w->probe || w->loopback) return false;
  if (!w->sim && w->nranks > 1) return false;
  return true;
}

static void enqueue_pipelined(Plan& p, cudaStream_t st);

void execute_plan(Plan* pp, float* const* grads, cudaStream_t st) {
  Plan& p = *pp;
  esp_world_s* w = p.w;
  const cudaStream_t cs = w->comm_stream;
  ESP_REQUIRE(!*const_cast<volatile unsigned int*>(w->wait_err_host), ESP_ERR_NCCL,
              "a peer's payload did not arrive within the wait timeout of an earlier call");
  if (!p.peers_ready && std::any_of(p.buckets.begin(), p.buckets.end(), [](const Bucket& b) { return b.fused; }))
    open_peers(p, cs);
  upload_dyn(p, grads, st);
  if (graphable(p)) {
    run_graphed(p, p.g_sync, st, [&](cudaStream_t s) {
      if (p.zero_bytes) ESP_CUDA(cudaMemsetAsync(p.zero, 0, p.zero_bytes, s));
      enqueue_pipelined(p, s);
    });
    for (auto* c : p.ctxs) c->step += 1;
    return;
  }
  if (p.zero_bytes) ESP_CUDA(cudaMemsetAsync(p.zero, 0, p.zero_bytes, st));
  const bool timing = w->timing;
  if (timing) {
    // serialised phases, events around each (a breakdown, not the pipelined time)
    const size_t nb = p.buckets.size();
    ESP_CUDA(cudaEventRecord(tev(w, 0), st));
    for (size_t i = 0; i < nb; ++i) {
      Bucket& b = p.buckets[i];
      cudaEvent_t e0 = tev(w, 1 + 6 * i), e1 = tev(w, 2 + 6 * i), e2 = tev(w, 3 + 6 * i);
      cudaEvent_t e3 = tev(w, 4 + 6 * i), m0 = tev(w, 5 + 6 * i), m1 = tev(w, 6 + 6 * i);
      ESP_CUDA(cudaEventRecord(e0, st));
      run_h1(p, b, st);
      ESP_CUDA(cudaEventRecord(e1, st));
      ESP_CUDA(cudaStreamWaitEvent(cs, e1, 0));
      ESP_CUDA(cudaEventRecord(m0, cs));
      ESP_CUDA(cudaEventRecord(m1, cs));
      run_comm(p, b, cs, m0, m1);
      ESP_CUDA(cudaEventRecord(e2, cs));
      ESP_CUDA(cudaStreamWaitEvent(st, e2, 0));
      run_h2(p, b, st);
      if (b.fused) ++b.epoch;
      ESP_CUDA(cudaEventRecord(e3, st));
    }
    ESP_CUDA(cudaEventRecord(tev(w, 1 + 6 * nb), st));
    ESP_CUDA(cudaEventSynchronize(tev(w, 1 + 6 * nb)));
    esp_timing_t t{};
    ESP_CUDA(cudaEventElapsedTime(&t.total_ms, tev(w, 0), tev(w, 1 + 6 * nb)));
    for (size_t i = 0; i < nb; ++i) {
      float a, bb, c, m;
      ESP_CUDA(cudaEventElapsedTime(&a, tev(w, 1 + 6 * i), tev(w, 2 + 6 * i)));
      ESP_CUDA(cudaEventElapsedTime(&bb, tev(w, 2 + 6 * i), tev(w, 3 + 6 * i)));
      ESP_CUDA(cudaEventElapsedTime(&c, tev(w, 3 + 6 * i), tev(w, 4 + 6 * i)));
      ESP_CUDA(cudaEventElapsedTime(&m, tev(w, 5 + 6 * i), tev(w, 6 + 6 * i)));
      t.h1_ms += a;
      t.comm_ms += bb - m;
      t.mid_ms += m;
      t.h2_ms += c;
    }
    w->last = t;
  } else {
    enqueue_pipelined(p, st);
  }
  for (auto* c : p.ctxs) c->step += 1;
}

// pipelined: h1(b+1) is issued before h2(b), so compression of the next
// bucket overlaps the collective of the previous one
static void enqueue_pipelined(Plan& p, cudaStream_t st) {
  esp_world_s* w = p.w;
  const cudaStream_t cs = w->comm_stream;
  ESP_CUDA(cudaEventRecord(w->ev_fork, st));
  ESP_CUDA(cudaStreamWaitEvent(cs, w->ev_fork, 0));
  const size_t nb = p.buckets.size();
  for (size_t i = 0; i <= nb; ++i) {
    if (i < nb) {
      Bucket& b = p.buckets[i];
      const cudaStream_t done = run_h1(p, b, st, nb > 1 ? w->fin_stream : nullptr);
      ESP_CUDA(cudaEventRecord(b.ev_h1, done));
      ESP_CUDA(cudaStreamWaitEvent(cs, b.ev_h1, 0));
      run_comm(p, b, cs, nullptr, nullptr);
      ESP_CUDA(cudaEventRecord(b.ev_comm, cs));
    }
    if (i >= 1) {
      Bucket& b = p.buckets[i - 1];
      ESP_CUDA(cudaStreamWaitEvent(st, b.ev_comm, 0));
      run_h2(p, b, st);
      if (b.fused) ++b.epoch;
    }
  }
}

// Loopback: the n worlds of one process on one GPU act as ranks 0..n-1 of a
// fused-collective job.  Their plans address each other's arenas directly (no
// IPC), and every kernel runs on one stream in an order that satisfies every
// dependency before it is launched: all ranks' h1, then stage 1 (pushes) of
// all ranks, stage 2, stage 3 (fused_stage), then all ranks' h2.  No kernel
// ever waits for a kernel launched after it, so nothing relies on concurrent
// residency on one GPU; a wrong job table leaves a counter short and its wait
// kernel reports a timeout.  This runs the real ranks' job tables, slot
// layouts, parities and counters for any n on a single GPU (tests).
void execute_loopback(const std::vector<Plan*>& plans, const std::vector<float* const*>& grads, cudaStream_t st) {
  const int n = (int)plans.size();
  for (Plan* p : plans)
    for (const Bucket& b : p->buckets)
      ESP_REQUIRE(b.fused, ESP_ERR_UNSUPPORTED,
                  "loopback worlds run the fused (byte-moving) routines only; NCCL-reduced buckets need a real world");
  for (Plan* p : plans) {
    ESP_REQUIRE(p->buckets.size() == plans[0]->buckets.size(), ESP_ERR_STATE, "ranks disagree on the bucketing");
    if (!p->peers_ready) {
      std::vector<unsigned char*> base(n);
      for (int q = 0; q < n; ++q) base[q] = plans[q]->arena.base;
      build_peer_tables(*p, base);
    }
  }
  for (int r = 0; r < n; ++r) {
    Plan& p = *plans[r];
    ESP_REQUIRE(!*const_cast<volatile unsigned int*>(p.w->wait_err_host), ESP_ERR_NCCL,
                "a payload did not arrive within the wait timeout of an earlier call");
    upload_dyn(p, grads[r], st);
    if (p.zero_bytes) ESP_CUDA(cudaMemsetAsync(p.zero, 0, p.zero_bytes, st));
  }
  for (size_t i = 0; i < plans[0]->buckets.size(); ++i) {
    for (int r = 0; r < n; ++r) run_h1(*plans[r], plans[r]->buckets[i], st);
    for (int stage = 1; stage <= 3; ++stage)
      for (int r = 0; r < n; ++r) fused_stage(*plans[r], plans[r]->buckets[i], stage, st, nullptr, nullptr);
    for (int r = 0; r < n; ++r) {
      run_h2(*plans[r], plans[r]->buckets[i], st);
      ++plans[r]->buckets[i].epoch;
    }
  }
  for (Plan* p : plans)
    for (auto* c : p->ctxs) c->step += 1;
}

void execute_compress(Plan* pp, const float* grad, void* payload, cudaStream_t st) {
  Plan& p = *pp;
  esp_ctx_s* c = p.ctxs[0];
  float* g = const_cast<float*>(grad);
  upload_dyn(p, &g, st);
  Bucket& b = p.buckets[0];
  auto body = [&](cudaStream_t s) {
    if (p.zero_bytes) ESP_CUDA(cudaMemsetAsync(p.zero, 0, p.zero_bytes, s));
    run_h1(p, b, s);
  };
  if (graphable(p)) run_graphed(p, p.g_compress, st, body);
  else body(st);
  for (int lr = 0; lr < p.w->nlocal; ++lr)
    ESP_CUDA(cudaMemcpyAsync((unsigned char*)payload + (size_t)lr * c->payload_bytes, b.send.at(lr),
                             c->payload_bytes, cudaMemcpyDeviceToDevice, st));
  c->step += 1;
}

}  // namespace esp
