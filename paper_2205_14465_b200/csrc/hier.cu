// Hierarchical communication ("the gradients
// are first aggregated among GPUs within one machine; they are then
// aggregated across machines; and the aggregated gradients are communicated
// within one machine again"; division schemes only for the
// intra-machine phases; reading R23).  n = m "machines" x g GPUs, emulated
// on one NVLink-5 box as groups of g consecutive ranks.  Per tensor:
//   A  intra-machine Reduce-scatter of the uncompressed tensor: every rank
//      packs its g shards (R10 partitions), pushes shard j to local GPU j
//      over NVLink and sums the g shards it receives in local-rank order
//      from +0 (/ g for MEAN) -- the machine's shard i;
//   B  inter-machine: the m GPUs holding shard i run the tensor's compressed
//      routine on it (h1 with EF -> Allgather / Alltoall-Allgather /
//      Gather-Broadcast -> h2), an ordinary plan of the `inter` world over
//      the shard ctxs, in place on the shard;
//   C  intra-machine Allgather: shard i goes to every local GPU, each unpacks
//      the g final shards into its gradient.
// A and C are push jobs with arrival counters over CUDA IPC of the plan's
// arena within the machine (call-parity receive buffers, as the flat fused
// collectives); B reuses the flat engine unchanged.
#include <algorithm>

#include "esp_internal.h"
#include "esp_kernels.h"

namespace esp {

struct HierPlan {
  esp_world_s* w = nullptr;
  std::vector<esp_ctx_s*> ctxs;
  std::vector<esp_ctx_s*> inner;            // the shard ctxs with a non-empty shard
  int g = 1, i = 0;                         // machine size, my local index
  size_t S = 0;                             // slot bytes: all tensors' (max-length) shards
  std::vector<size_t> coff;                 // tensor offset within a slot
  std::vector<uint32_t> L;                  // tensor shard length (max)
  Arena arena;
  // peer-visible section first (identical layout everywhere)
  size_t recvA_off = 0, recvC_off = 0, cnt_off = 0;
  unsigned char *sendA = nullptr, *mid = nullptr;
  uint64_t* dyn = nullptr;                  // device: gradient pointers of the call
  uint64_t* mid_word = nullptr;             // device: the mid buffer's base (h2's output pointer)
  uint64_t* dyn_host = nullptr;             // pinned staging of the pointers
  cudaEvent_t dyn_ev = nullptr;
  bool dyn_pending = false;
  // tables
  SegH1* pack = nullptr; uint32_t* pack_units = nullptr; int npack_units = 0;
  SegH2* sum = nullptr; uint32_t* sum_units = nullptr; int nsum_units = 0;
  const unsigned char** sum_pieces[2] = {nullptr, nullptr};
  SegH2* unpack = nullptr; uint32_t* unpack_units = nullptr; int nunpack_units = 0;
  const unsigned char** unpack_pieces[2] = {nullptr, nullptr};
  PushJob* pushA = nullptr; int npushA = 0;
  PushJob* pushC = nullptr; int npushC = 0;
  uint64_t targetA = 0, targetC = 0;        // arrivals per call
  unsigned char** dstA = nullptr;           // device [2][g]: my slot in every local GPU's recvA / recvC
  unsigned char** dstC = nullptr;
  unsigned long long** cntA = nullptr;      // device [2][g]: their counters
  unsigned long long** cntC = nullptr;
  unsigned long long* my_cnt = nullptr;     // [A par0, A par1, C par0, C par1]
  std::vector<void*> peer_bases;            // IPC-opened arenas of the machine's other GPUs
  bool peers_ready = false;
  uint64_t epoch = 0;
  std::vector<float*> inner_grads;          // the shards in `mid`, one per inner ctx
  std::vector<void*> dev_allocs;
  ~HierPlan() {
    for (void* p : peer_bases)
      if (p) cudaIpcCloseMemHandle(p);
    for (void* p : dev_allocs) cudaFree(p);
    if (dyn_host) cudaFreeHost(dyn_host);
    if (dyn_ev) cudaEventDestroy(dyn_ev);
  }
};

namespace {

uint32_t shard_lo(uint64_t N, int g, int j) {
  const uint64_t Lmax = partition_len(N, g);
  return (uint32_t)std::min<uint64_t>(N, (uint64_t)j * (g == 1 ? N : Lmax));
}
uint32_t shard_hi(uint64_t N, int g, int j) {
  if (g == 1) return (uint32_t)N;
  return (uint32_t)std::min<uint64_t>(N, (uint64_t)shard_lo(N, g, j) + partition_len(N, g));
}

template <class T>
T* upload(HierPlan& h, const std::vector<T>& v) {
  T* d = nullptr;
  ESP_CUDA(cudaMalloc(&d, sizeof(T) * std::max<size_t>(1, v.size())));
  if (!v.empty()) ESP_CUDA(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  h.dev_allocs.push_back(d);
  return d;
}

void add_jobs(std::vector<PushJob>& v, size_t src_off, size_t bytes, int d) {
  for (size_t c = 0; c < bytes; c += kPushChunk)
    v.push_back(PushJob{src_off + c, c, (uint32_t)std::min<size_t>(kPushChunk, bytes - c), (uint32_t)d});
}

HierPlan* build(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs) {
  auto h = std::make_unique<HierPlan>();
  h->w = w;
  h->ctxs = ctxs;
  const int g = w->hier_g, i = w->rank % g;
  h->g = g;
  h->i = i;
  const size_t nt = ctxs.size();
  for (esp_ctx_s* c : ctxs) {
    h->coff.push_back(h->S);
    h->L.push_back((uint32_t)partition_len(c->N, g));
    h->S += round_up(4ull * h->L.back(), 16);
    if (c->inner) h->inner.push_back(c->inner);
  }
  // arena: [recvA 2 x g x S][recvC 2 x g x S][counters] | [sendA g x S][mid S][dyn][mid word]
  Arena& a = h->arena;
  h->recvA_off = a.reserve(2ull * g * h->S);
  h->recvC_off = a.reserve(2ull * g * h->S);
  h->cnt_off = a.reserve(256);
  const size_t sendA_off = a.reserve((size_t)g * h->S);
  const size_t mid_off = a.reserve(h->S);
  const size_t dyn_off = a.reserve(8 * std::max<size_t>(1, nt));
  const size_t word_off = a.reserve(8);
  a.alloc();
  ESP_CUDA(cudaMemset(a.base, 0, a.size));
  unsigned char* B = a.base;
  h->sendA = B + sendA_off;
  h->mid = B + mid_off;
  h->dyn = reinterpret_cast<uint64_t*>(B + dyn_off);
  h->mid_word = reinterpret_cast<uint64_t*>(B + word_off);
  const uint64_t midp = (uint64_t)(uintptr_t)h->mid;
  ESP_CUDA(cudaMemcpy(h->mid_word, &midp, 8, cudaMemcpyHostToDevice));
  h->my_cnt = reinterpret_cast<unsigned long long*>(B + h->cnt_off);
  ESP_CUDA(cudaMallocHost(&h->dyn_host, 8 * std::max<size_t>(1, nt)));
  ESP_CUDA(cudaEventCreateWithFlags(&h->dyn_ev, cudaEventDisableTiming));
  const float divisor = ctxs[0]->cfg.reduce == ESP_MEAN ? (float)g : 1.0f;

  // A: pack every (tensor, shard j) into sendA slot j
  std::vector<SegH1> pack;
  std::vector<uint32_t> pack_units;
  for (size_t t = 0; t < nt; ++t)
    for (int j = 0; j < g; ++j) {
      const uint32_t lo = shard_lo(ctxs[t]->N, g, j), hi = shard_hi(ctxs[t]->N, g, j);
      if (hi == lo) continue;
      SegH1 s{};
      s.gptr = h->dyn + t;
      s.goff = lo;
      s.chunk = h->sendA + (size_t)j * h->S + h->coff[t];
      s.n = hi - lo;
      s.nunits = div_up(s.n, kUnit);
      s.unit0 = (uint32_t)pack_units.size();
      for (uint32_t u = 0; u < s.nunits; ++u) pack_units.push_back((uint32_t)pack.size());
      pack.push_back(s);
    }
  h->pack = upload(*h, pack);
  h->pack_units = upload(*h, pack_units);
  h->npack_units = (int)pack_units.size();
  // A: slot j to local GPU j (its recvA slot i), then the sum of the g slots
  std::vector<PushJob> pa, pc;
  for (int j = 0; j < g; ++j)
    if (j != i) add_jobs(pa, (size_t)j * h->S, h->S, j);
  for (int j = 0; j < g; ++j)
    if (j != i) add_jobs(pc, 0, h->S, j);
  h->pushA = upload(*h, pa);
  h->npushA = (int)pa.size();
  h->pushC = upload(*h, pc);
  h->npushC = (int)pc.size();
  const uint64_t J = div_up(h->S, kPushChunk);
  h->targetA = h->targetC = (uint64_t)(g - 1) * J;
  std::vector<SegH2> sum;
  std::vector<uint32_t> sum_units;
  std::vector<const unsigned char*> sp[2];
  for (size_t t = 0; t < nt; ++t) {
    const uint32_t lo = shard_lo(ctxs[t]->N, g, i), hi = shard_hi(ctxs[t]->N, g, i);
    if (hi == lo) continue;
    SegH2 s{};
    s.optr = h->mid_word;
    s.ooff = h->coff[t] / 4;
    s.n = hi - lo;
    s.npieces = (uint32_t)g;
    s.piece0 = (uint32_t)sp[0].size();
    s.divisor = divisor;
    for (int j = 0; j < g; ++j)   // local-rank order; my own shard from sendA
      for (int par = 0; par < 2; ++par)
        sp[par].push_back(j == i ? h->sendA + (size_t)i * h->S + h->coff[t]
                                 : B + h->recvA_off + ((size_t)par * g + j) * h->S + h->coff[t]);
    s.nunits = div_up(s.n, kUnit);
    s.unit0 = (uint32_t)sum_units.size();
    for (uint32_t u = 0; u < s.nunits; ++u) sum_units.push_back((uint32_t)sum.size());
    sum.push_back(s);
  }
  h->sum = upload(*h, sum);
  h->sum_units = upload(*h, sum_units);
  h->nsum_units = (int)sum_units.size();
  for (int par = 0; par < 2; ++par) h->sum_pieces[par] = upload(*h, sp[par]);
  // C: every (tensor, shard j) from recvC slot j (mine from mid) into the gradient
  std::vector<SegH2> up;
  std::vector<uint32_t> up_units;
  std::vector<const unsigned char*> upp[2];
  for (size_t t = 0; t < nt; ++t)
    for (int j = 0; j < g; ++j) {
      const uint32_t lo = shard_lo(ctxs[t]->N, g, j), hi = shard_hi(ctxs[t]->N, g, j);
      if (hi == lo) continue;
      SegH2 s{};
      s.optr = h->dyn + t;
      s.ooff = lo;
      s.n = hi - lo;
      s.npieces = 1;
      s.piece0 = (uint32_t)upp[0].size();
      s.divisor = 1.0f;
      for (int par = 0; par < 2; ++par)
        upp[par].push_back(j == i ? h->mid + h->coff[t] : B + h->recvC_off + ((size_t)par * g + j) * h->S + h->coff[t]);
      s.nunits = div_up(s.n, kUnit);
      s.unit0 = (uint32_t)up_units.size();
      for (uint32_t u = 0; u < s.nunits; ++u) up_units.push_back((uint32_t)up.size());
      up.push_back(s);
    }
  h->unpack = upload(*h, up);
  h->unpack_units = upload(*h, up_units);
  h->nunpack_units = (int)up_units.size();
  for (int par = 0; par < 2; ++par) h->unpack_pieces[par] = upload(*h, upp[par]);
  // B: the shards in `mid` are the inner ctxs' gradients
  for (size_t t = 0; t < nt; ++t)
    if (ctxs[t]->inner) h->inner_grads.push_back(reinterpret_cast<float*>(h->mid + h->coff[t]));
  return h.release();
}

// my slot / counters in every local GPU's arena, per parity ([par][j])
void peer_tables(HierPlan& h, const std::vector<unsigned char*>& base) {
  const int g = h.g;
  std::vector<unsigned char*> da(2 * g), dc(2 * g);
  std::vector<unsigned long long*> ca(2 * g), cc(2 * g);
  for (int par = 0; par < 2; ++par)
    for (int j = 0; j < g; ++j) {
      da[par * g + j] = base[j] + h.recvA_off + ((size_t)par * g + h.i) * h.S;
      dc[par * g + j] = base[j] + h.recvC_off + ((size_t)par * g + h.i) * h.S;
      unsigned long long* c = reinterpret_cast<unsigned long long*>(base[j] + h.cnt_off);
      ca[par * g + j] = c + par;
      cc[par * g + j] = c + 2 + par;
    }
  h.dstA = upload(h, da);
  h.dstC = upload(h, dc);
  h.cntA = upload(h, ca);
  h.cntC = upload(h, cc);
  h.peers_ready = true;
}

// the machine's arenas over CUDA IPC (collective over the intra world)
void open_peers(HierPlan& h, cudaStream_t st) {
  esp_world_s* in = h.w->intra;
  const int g = h.g;
  cudaIpcMemHandle_t mine;
  ESP_CUDA(cudaIpcGetMemHandle(&mine, h.arena.base));
  unsigned char* d = nullptr;
  ESP_CUDA(cudaMalloc(&d, sizeof(mine) * (g + 1)));
  ESP_CUDA(cudaMemcpy(d + sizeof(mine) * g, &mine, sizeof(mine), cudaMemcpyHostToDevice));
  ESP_NCCL(ncclAllGather(d + sizeof(mine) * g, d, sizeof(mine), ncclUint8, in->comm, st));
  std::vector<cudaIpcMemHandle_t> all(g);
  ESP_CUDA(cudaStreamSynchronize(st));
  ESP_CUDA(cudaMemcpy(all.data(), d, sizeof(mine) * g, cudaMemcpyDeviceToHost));
  cudaFree(d);
  std::vector<unsigned char*> base(g);
  h.peer_bases.assign(g, nullptr);
  for (int j = 0; j < g; ++j) {
    if (j == h.i) {
      base[j] = h.arena.base;
      continue;
    }
    void* p = nullptr;
    ESP_CUDA(cudaIpcOpenMemHandle(&p, all[j], cudaIpcMemLazyEnablePeerAccess));
    h.peer_bases[j] = p;
    base[j] = static_cast<unsigned char*>(p);
  }
  peer_tables(h, base);
}

void upload_dyn(HierPlan& h, float* const* grads, cudaStream_t st) {
  if (h.dyn_pending) ESP_CUDA(cudaEventSynchronize(h.dyn_ev));
  for (size_t t = 0; t < h.ctxs.size(); ++t) h.dyn_host[t] = (uint64_t)(uintptr_t)grads[t];
  ESP_CUDA(cudaMemcpyAsync(h.dyn, h.dyn_host, 8 * h.ctxs.size(), cudaMemcpyHostToDevice, st));
  ESP_CUDA(cudaEventRecord(h.dyn_ev, st));
  h.dyn_pending = true;
}

// the stages of one call; across the machine's ranks stage s only depends on
// stages < s of the others (the loopback executor runs them rank by rank)
void stage_A_push(HierPlan& h, cudaStream_t st) {
  const int par = (int)(h.epoch & 1);
  launch_pack(h.pack, h.pack_units, h.npack_units, st);
  launch_push(h.pushA, h.npushA, h.sendA, h.dstA + par * h.g, h.cntA + par * h.g, st);
  const uint64_t v = 4ull * (h.S / 4) * (h.g - 1);   // logical: my g - 1 shards out, theirs in
  count_coll(h.w, 0, ESP_OP_REDUCESCATTER, v, v);
  h.w->counters[0].pushed += v;
}
void stage_A_sum(HierPlan& h, cudaStream_t st) {
  const int par = (int)(h.epoch & 1);
  launch_wait_arrivals(h.my_cnt + par, ((h.epoch >> 1) + 1) * h.targetA, h.w->wait_err, h.w->wait_timeout_ns, st);
  launch_h2_dense(h.sum, h.sum_units, h.nsum_units, h.sum_pieces[par], st);
}
void stage_C_push(HierPlan& h, cudaStream_t st) {
  const int par = (int)(h.epoch & 1);
  launch_push(h.pushC, h.npushC, h.mid, h.dstC + par * h.g, h.cntC + par * h.g, st);
  const uint64_t v = 4ull * (h.S / 4) * (h.g - 1);
  count_coll(h.w, 0, ESP_OP_ALLGATHER, v, v);
  h.w->counters[0].pushed += v;
}
void stage_C_unpack(HierPlan& h, cudaStream_t st) {
  const int par = (int)(h.epoch & 1);
  launch_wait_arrivals(h.my_cnt + 2 + par, ((h.epoch >> 1) + 1) * h.targetC, h.w->wait_err, h.w->wait_timeout_ns,
                       st);
  launch_h2_dense(h.unpack, h.unpack_units, h.nunpack_units, h.unpack_pieces[par], st);
}

HierPlan* find_or_build(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs) {
  for (HierPlan* p : w->hplans)
    if (p->ctxs == ctxs) return p;
  w->hplans.push_back(build(w, ctxs));
  return w->hplans.back();
}

}  // namespace

void execute_hier(esp_world_s* w, const std::vector<esp_ctx_s*>& ctxs, float* const* grads, cudaStream_t st) {
  ESP_REQUIRE(!*const_cast<volatile unsigned int*>(w->wait_err_host), ESP_ERR_NCCL,
              "a peer's payload did not arrive within the wait timeout of an earlier call");
  HierPlan& h = *find_or_build(w, ctxs);
  if (!h.peers_ready) open_peers(h, st);
  upload_dyn(h, grads, st);
  stage_A_push(h, st);
  stage_A_sum(h, st);
  if (!h.inner.empty()) {
    esp_world_s* x = w->inter;
    Plan* p = get_plan(x, h.inner);
    execute_plan(p, h.inner_grads.data(), st);
  }
  stage_C_push(h, st);
  stage_C_unpack(h, st);
  ++h.epoch;
  for (esp_ctx_s* c : ctxs) c->step += 1;
}

void execute_hier_loopback(const std::vector<esp_world_s*>& ws, const std::vector<std::vector<esp_ctx_s*>>& ctxs,
                           const std::vector<float* const*>& grads, cudaStream_t st) {
  const int n = (int)ws.size(), g = ws[0]->hier_g, m = n / g;
  std::vector<HierPlan*> hp(n);
  for (int r = 0; r < n; ++r) hp[r] = find_or_build(ws[r], ctxs[r]);
  for (int r = 0; r < n; ++r)
    if (!hp[r]->peers_ready) {   // the machine's arenas, by plain pointers
      std::vector<unsigned char*> base(g);
      const int a = r / g;
      for (int j = 0; j < g; ++j) base[j] = hp[a * g + j]->arena.base;
      peer_tables(*hp[r], base);
    }
  for (int r = 0; r < n; ++r) {
    ESP_REQUIRE(!*const_cast<volatile unsigned int*>(ws[r]->wait_err_host), ESP_ERR_NCCL,
                "a payload did not arrive within the wait timeout of an earlier call");
    upload_dyn(*hp[r], grads[r], st);
  }
  for (int r = 0; r < n; ++r) stage_A_push(*hp[r], st);
  for (int r = 0; r < n; ++r) stage_A_sum(*hp[r], st);
  for (int i = 0; i < g; ++i) {   // the inter-machine group of local index i
    if (hp[i]->inner.empty()) continue;
    std::vector<Plan*> plans(m);
    std::vector<float* const*> gr(m);
    for (int a = 0; a < m; ++a) {
      HierPlan& h = *hp[a * g + i];
      plans[a] = get_plan(ws[a * g + i]->inter, h.inner);
      gr[a] = h.inner_grads.data();
    }
    if (m == 1) execute_plan(plans[0], gr[0], st);
    else execute_loopback(plans, gr, st);
  }
  for (int r = 0; r < n; ++r) stage_C_push(*hp[r], st);
  for (int r = 0; r < n; ++r) stage_C_unpack(*hp[r], st);
  for (int r = 0; r < n; ++r) {
    ++hp[r]->epoch;
    for (esp_ctx_s* c : ctxs[r]) c->step += 1;
  }
}

void clear_hier_plans(esp_world_s* w) {
  if (!w->hplans.empty()) cudaDeviceSynchronize();
  for (HierPlan* p : w->hplans) delete p;
  w->hplans.clear();
}

void drop_hier_plans_with(esp_world_s* w, esp_ctx_s* c) {
  auto& v = w->hplans;
  for (auto it = v.begin(); it != v.end();) {
    if (std::find((*it)->ctxs.begin(), (*it)->ctxs.end(), c) != (*it)->ctxs.end()) {
      cudaDeviceSynchronize();
      delete *it;
      it = v.erase(it);
    } else {
      ++it;
    }
  }
}

}  // namespace esp
