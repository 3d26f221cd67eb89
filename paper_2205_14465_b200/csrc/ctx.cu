// Per-tensor contexts (the paper's per-tensor compression option c_j, P:1133 /
// P:1169, restricted to flat GPU compression) and the h1 / h2 / sync entry
// points of the C ABI.
#include <algorithm>
#include <cmath>

#include "esp_internal.h"
#include "esp_kernels.h"

using namespace esp;

namespace {

constexpr uint64_t kStateMagic = 0x4553505354415445ull;   // "ESPSTATE"

struct StateHeader {
  uint64_t magic, step, numel, r2_len, nlocal;
};

void check_cfg(const esp_compressor_cfg_t* cfg) {
  ESP_REQUIRE(cfg, ESP_ERR_INVALID_ARG, "cfg is NULL");
  ESP_REQUIRE(cfg->kind >= ESP_NONE && cfg->kind <= ESP_ONEBIT, ESP_ERR_INVALID_ARG, "bad compressor kind");
  ESP_REQUIRE(cfg->reduce == ESP_MEAN || cfg->reduce == ESP_SUM, ESP_ERR_INVALID_ARG, "bad reduce mode");
  ESP_REQUIRE(cfg->process >= 0 && cfg->process <= 2, ESP_ERR_INVALID_ARG, "process must be 0, 1 or 2");
  ESP_REQUIRE(cfg->momentum >= 0.0 && cfg->momentum < 1.0, ESP_ERR_INVALID_ARG, "momentum must be in [0, 1)");
  if (cfg->momentum != 0.0)
    ESP_REQUIRE((cfg->kind == ESP_DGC || cfg->kind == ESP_TOPK) && cfg->error_feedback, ESP_ERR_INVALID_ARG,
                "momentum correction needs DGC/TOPK with error feedback (R20)");
  if (is_sparse(cfg->kind))
    ESP_REQUIRE(cfg->ratio > 0.0 && cfg->ratio <= 1.0, ESP_ERR_INVALID_ARG, "ratio must be in (0, 1]");
  ESP_REQUIRE(cfg->dgc_approx == 0 || cfg->dgc_approx == 1, ESP_ERR_INVALID_ARG, "dgc_approx must be 0 or 1");
  ESP_REQUIRE(!cfg->dgc_approx || cfg->kind == ESP_DGC, ESP_ERR_INVALID_ARG,
              "the approximate-count mode is DGC's (R22)");
  ESP_REQUIRE(cfg->dgc_sample_rate >= 0.0 && cfg->dgc_sample_rate <= 1.0, ESP_ERR_INVALID_ARG,
              "dgc_sample_rate must be in [0, 1]");
}

void check_ptr16(const void* p, const char* what) {
  ESP_REQUIRE(p, ESP_ERR_INVALID_ARG, std::string(what) + " is NULL");
  ESP_REQUIRE(((uintptr_t)p & 15) == 0, ESP_ERR_INVALID_ARG, std::string(what) + " is not 16-byte aligned");
}

// gradients of esp_sync / esp_sync_many: 4-byte alignment suffices (tensors that
// are not 16-byte aligned take the guarded-load paths of the kernels; e.g. the
// per-parameter views of a DDP gradient bucket)
void check_ptr4(const void* p, const char* what) {
  ESP_REQUIRE(p, ESP_ERR_INVALID_ARG, std::string(what) + " is NULL");
  ESP_REQUIRE(((uintptr_t)p & 3) == 0, ESP_ERR_INVALID_ARG, std::string(what) + " is not 4-byte aligned");
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

esp_status_t esp_ctx_create(esp_world_t w, const esp_compressor_cfg_t* cfg, int routine, uint64_t tensor_id,
                            size_t numel, esp_ctx_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && out, ESP_ERR_INVALID_ARG, "null argument");
  check_cfg(cfg);
  ESP_REQUIRE(routine >= ESP_ALLREDUCE && routine <= ESP_REDUCE_BROADCAST, ESP_ERR_INVALID_ARG, "bad routine");
  ESP_REQUIRE(numel >= 1, ESP_ERR_INVALID_ARG, "numel must be >= 1");
  ESP_REQUIRE(numel < (1ull << 31), ESP_ERR_TOO_LARGE, "numel >= 2^31 (uint32 indices, R18)");
  ESP_REQUIRE(pair_legal(*cfg, routine), ESP_ERR_UNSUPPORTED,
              "illegal (compressor, routine) pair (P:1064-1065, P:1073)");
  ESP_CUDA(cudaSetDevice(w->dev));
  if (w->hier_g > 0) {
    // hierarchical world (R23): the tensor's state is that of this rank's
    // shard, a ctx of the inter-machine world (tensor id * 4096 + shard)
    ESP_REQUIRE(cfg->kind != ESP_NONE && routine != ESP_ALLREDUCE, ESP_ERR_UNSUPPORTED,
                "hierarchical sync compresses the inter-machine phase: a compressed kind with Allgather, "
                "Alltoall/Allgather or Gather/Broadcast");
    const int g = w->hier_g, i = w->rank % g;
    const uint64_t L = partition_len(numel, g);
    const uint64_t lo = g == 1 ? 0 : std::min<uint64_t>(numel, (uint64_t)i * L);
    const uint64_t hi = g == 1 ? numel : std::min<uint64_t>(numel, lo + L);
    auto c = std::make_unique<esp_ctx_s>();
    c->w = w;
    c->cfg = *cfg;
    c->routine = routine;
    c->tensor_id = tensor_id;
    c->N = numel;
    if (hi > lo) {
      esp_ctx_t in = nullptr;
      const esp_status_t s = esp_ctx_create(w->inter, cfg, routine, tensor_id * 4096 + (uint64_t)i, hi - lo, &in);
      if (s != ESP_OK) return s;
      c->inner = in;
      c->payload_bytes = in->payload_bytes;
    }
    w->ctxs.insert(c.get());
    *out = c.release();
    return ESP_OK;
  }
  auto c = std::make_unique<esp_ctx_s>();
  c->w = w;
  c->cfg = *cfg;
  c->routine = routine;
  c->tensor_id = tensor_id;
  c->N = numel;
  const int n = w->nranks, nl = w->nlocal;
  c->P = cfg->kind == ESP_NONE ? 1 : nparts_of(routine, n);
  const uint64_t L = partition_len(numel, c->P);
  for (int p = 0; p < c->P; ++p) {
    uint64_t lo = c->P == 1 ? 0 : std::min<uint64_t>(numel, (uint64_t)p * L);
    uint64_t hi = c->P == 1 ? numel : std::min<uint64_t>(numel, lo + L);
    c->plo.push_back((uint32_t)lo);
    c->phi.push_back((uint32_t)hi);
    c->pk.push_back(k_of(hi - lo, cfg->ratio));
  }
  c->chunk_bytes = chunk_bytes_of(*cfg, numel, c->P, &c->kpad);
  c->payload_bytes = c->chunk_bytes * c->P;
  c->hash_base = host_splitmix64(host_splitmix64(cfg->seed) ^ tensor_id);
  if (cfg->kind != ESP_NONE) {
    ESP_CUDA(cudaMalloc(&c->r, sizeof(float) * numel * nl));
    ESP_CUDA(cudaMemset(c->r, 0, sizeof(float) * numel * nl));
    ESP_CUDA(cudaMalloc(&c->lazy, sizeof(float) * 2 * c->P * nl));
    ESP_CUDA(cudaMemset(c->lazy, 0, sizeof(float) * 2 * c->P * nl));
  }
  if (cfg->momentum != 0.0) {
    ESP_CUDA(cudaMalloc(&c->u, sizeof(float) * numel * nl));
    ESP_CUDA(cudaMemset(c->u, 0, sizeof(float) * numel * nl));
  }
  if (mid_scheme(*cfg, routine)) {
    c->r2_len = routine == ESP_ALLTOALL_ALLGATHER ? L : numel;
    ESP_CUDA(cudaMalloc(&c->r2, sizeof(float) * c->r2_len * nl));
    ESP_CUDA(cudaMemset(c->r2, 0, sizeof(float) * c->r2_len * nl));
    if (is_quant(cfg->kind)) {
      ESP_CUDA(cudaMalloc(&c->lazy2, sizeof(float) * 2 * nl));
      ESP_CUDA(cudaMemset(c->lazy2, 0, sizeof(float) * 2 * nl));
    }
  }
  if ((cfg->kind == ESP_DGC || cfg->kind == ESP_TOPK) && (cfg->error_feedback || cfg->momentum != 0.0)) {
    // deferred EF zeroing records: capacity for ~ e + 4 sqrt(e) + 8 selected
    // per 4096-element tile (e = 4096 ratio); a fuller tile zeroes the rest directly
    const double e = 4096.0 * std::min(1.0, cfg->ratio), want = e + 4.0 * std::sqrt(e) + 8.0;
    c->zcap = want <= 31.0 ? 32u : want <= 63.0 ? 64u : 128u;
    for (int p = 0; p < c->P; ++p) {
      c->zrec_part.push_back(c->zrec_stride);
      c->zrec_stride += (size_t)div_up(c->phi[p] - c->plo[p], kDgcTile) * c->zcap;
    }
    ESP_CUDA(cudaMalloc(&c->zrec, 2 * std::max<size_t>(1, c->zrec_stride * nl)));
    ESP_CUDA(cudaMemset(c->zrec, 0, 2 * std::max<size_t>(1, c->zrec_stride * nl)));
    if (c->r2 && cfg->error_feedback) {
      c->zrec2_stride = (size_t)div_up(c->r2_len, kDgcTile) * c->zcap;
      ESP_CUDA(cudaMalloc(&c->zrec2, 2 * std::max<size_t>(1, c->zrec2_stride * nl)));
      ESP_CUDA(cudaMemset(c->zrec2, 0, 2 * std::max<size_t>(1, c->zrec2_stride * nl)));
    }
  }
  w->ctxs.insert(c.get());
  *out = c.release();
  ESP_API_END
}

esp_status_t esp_ctx_destroy(esp_ctx_t c) {
  ESP_API_BEGIN
  ESP_REQUIRE(c, ESP_ERR_INVALID_ARG, "ctx is NULL");
  cudaSetDevice(c->w->dev);
  drop_plans_with(c->w, c);
  drop_hier_plans_with(c->w, c);
  cudaDeviceSynchronize();
  if (c->inner) esp_ctx_destroy(c->inner);
  cudaFree(c->r);
  cudaFree(c->lazy);
  cudaFree(c->r2);
  cudaFree(c->lazy2);
  cudaFree(c->u);
  cudaFree(c->zrec);
  cudaFree(c->zrec2);
  if (c->dec.d) cudaFree(c->dec.d);
  if (c->dec.acc) cudaFree(c->dec.acc);
  if (c->dec.h) cudaFreeHost(c->dec.h);
  if (c->dec.ev) cudaEventDestroy(c->dec.ev);
  c->w->ctxs.erase(c);
  delete c;
  ESP_API_END
}

esp_status_t esp_ctx_payload_bytes(esp_ctx_t c, size_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(c && out, ESP_ERR_INVALID_ARG, "null argument");
  *out = c->payload_bytes;
  ESP_API_END
}

// valid length of local rank lr's second residual
static uint64_t r2_valid(esp_ctx_t c, int lr) {
  if (!c->r2) return 0;
  const int j = c->w->sim ? lr : c->w->rank;
  if (c->routine == ESP_ALLTOALL_ALLGATHER) return c->phi[j] - c->plo[j];
  return j == 0 ? c->N : 0;
}

// The pending deferred EF zeroing of every segment of c applied to r / u / r2
// in memory (records cleared): the state is then the plain residual.
static void apply_zrec(esp_ctx_s* c) {
  const int nl = c->w->nlocal;
  for (int lr = 0; lr < nl; ++lr) {
    if (c->zrec)
      for (int p = 0; p < c->P; ++p) {
        const size_t off = (size_t)lr * c->N + c->plo[p];
        launch_dgc_zrec_apply(c->cfg.error_feedback ? c->r + off : nullptr, c->u ? c->u + off : nullptr,
                              c->zrec + (size_t)lr * c->zrec_stride + c->zrec_part[p], c->zcap, c->phi[p] - c->plo[p], 0);
      }
    if (c->zrec2)
      launch_dgc_zrec_apply(c->r2 + (size_t)lr * c->r2_len, nullptr, c->zrec2 + (size_t)lr * c->zrec2_stride, c->zcap,
                            (uint32_t)c->r2_len, 0);
  }
  ESP_CUDA(cudaGetLastError());
  ESP_CUDA(cudaDeviceSynchronize());
}

esp_status_t esp_ctx_get_state(esp_ctx_t c, void* host_buf, size_t* nbytes) {
  ESP_API_BEGIN
  ESP_REQUIRE(c && nbytes, ESP_ERR_INVALID_ARG, "null argument");
  if (c->w->hier_g > 0) {   // the rank's shard
    ESP_REQUIRE(c->inner, ESP_ERR_STATE, "this rank's shard of the tensor is empty");
    return esp_ctx_get_state(c->inner, host_buf, nbytes);
  }
  const int nl = c->w->nlocal;
  const size_t need = sizeof(StateHeader) + (size_t)nl * 4 * (c->N + c->r2_len);
  if (!host_buf) {
    *nbytes = need;
    return ESP_OK;
  }
  ESP_REQUIRE(*nbytes >= need, ESP_ERR_INVALID_ARG, "state buffer too small");
  ESP_CUDA(cudaSetDevice(c->w->dev));
  ESP_CUDA(cudaDeviceSynchronize());
  apply_zrec(c);
  StateHeader h{kStateMagic, c->step, c->N, c->r2_len, (uint64_t)nl};
  std::memcpy(host_buf, &h, sizeof(h));
  float* out = reinterpret_cast<float*>((unsigned char*)host_buf + sizeof(h));
  float* tmp = nullptr;
  ESP_CUDA(cudaMalloc(&tmp, sizeof(float) * std::max<uint64_t>(1, std::max(c->N, c->r2_len))));
  const int kk = c->cfg.kind == ESP_EFSIGNSGD ? K_EFSIGN : K_ONEBIT;
  for (int lr = 0; lr < nl; ++lr) {
    float* dst = out + (size_t)lr * (c->N + c->r2_len);
    if (!c->r) {
      std::memset(dst, 0, 4 * c->N);
    } else if (is_quant(c->cfg.kind)) {
      for (int p = 0; p < c->P; ++p) {
        const uint32_t lo = c->plo[p], len = c->phi[p] - c->plo[p];
        launch_sign_materialize(kk, c->r + (size_t)lr * c->N + lo, c->lazy + ((size_t)lr * c->P + p) * 2,
                                tmp + lo, len, 0);
      }
      ESP_CUDA(cudaMemcpy(dst, tmp, 4 * c->N, cudaMemcpyDeviceToHost));
    } else {
      ESP_CUDA(cudaMemcpy(dst, c->r + (size_t)lr * c->N, 4 * c->N, cudaMemcpyDeviceToHost));
    }
    float* dst2 = dst + c->N;
    std::memset(dst2, 0, 4 * c->r2_len);
    const uint64_t v = r2_valid(c, lr);
    if (v && c->lazy2) {
      launch_sign_materialize(kk, c->r2 + (size_t)lr * c->r2_len, c->lazy2 + (size_t)lr * 2, tmp, (uint32_t)v, 0);
      ESP_CUDA(cudaMemcpy(dst2, tmp, 4 * v, cudaMemcpyDeviceToHost));
    } else if (v) {
      ESP_CUDA(cudaMemcpy(dst2, c->r2 + (size_t)lr * c->r2_len, 4 * v, cudaMemcpyDeviceToHost));
    }
  }
  cudaFree(tmp);
  *nbytes = need;
  ESP_API_END
}

esp_status_t esp_ctx_set_state(esp_ctx_t c, const void* host_buf, size_t nbytes) {
  ESP_API_BEGIN
  ESP_REQUIRE(c && host_buf, ESP_ERR_INVALID_ARG, "null argument");
  if (c->w->hier_g > 0) {
    ESP_REQUIRE(c->inner, ESP_ERR_STATE, "this rank's shard of the tensor is empty");
    return esp_ctx_set_state(c->inner, host_buf, nbytes);
  }
  StateHeader h;
  ESP_REQUIRE(nbytes >= sizeof(h), ESP_ERR_INVALID_ARG, "state blob too small");
  std::memcpy(&h, host_buf, sizeof(h));
  const int nl = c->w->nlocal;
  ESP_REQUIRE(h.magic == kStateMagic && h.numel == c->N && h.r2_len == c->r2_len && h.nlocal == (uint64_t)nl,
              ESP_ERR_STATE, "state blob does not match this ctx");
  ESP_REQUIRE(nbytes >= sizeof(h) + (size_t)nl * 4 * (c->N + c->r2_len), ESP_ERR_INVALID_ARG, "blob truncated");
  ESP_CUDA(cudaSetDevice(c->w->dev));
  ESP_CUDA(cudaDeviceSynchronize());
  apply_zrec(c);   // u's pending zeros stay applied; r / r2 are overwritten below
  const float* in = reinterpret_cast<const float*>((const unsigned char*)host_buf + sizeof(h));
  for (int lr = 0; lr < nl; ++lr) {
    const float* src = in + (size_t)lr * (c->N + c->r2_len);
    // the true residual with a zero scale pair is its own lazy representation
    if (c->r) ESP_CUDA(cudaMemcpy(c->r + (size_t)lr * c->N, src, 4 * c->N, cudaMemcpyHostToDevice));
    if (c->r2) ESP_CUDA(cudaMemcpy(c->r2 + (size_t)lr * c->r2_len, src + c->N, 4 * c->r2_len, cudaMemcpyHostToDevice));
  }
  if (c->lazy) ESP_CUDA(cudaMemset(c->lazy, 0, sizeof(float) * 2 * c->P * nl));
  if (c->lazy2) ESP_CUDA(cudaMemset(c->lazy2, 0, sizeof(float) * 2 * nl));
  c->step = h.step;
  ESP_API_END
}

esp_status_t esp_ctx_get_momentum(esp_ctx_t c, float* host, size_t count) {
  ESP_API_BEGIN
  ESP_REQUIRE(c && host, ESP_ERR_INVALID_ARG, "null argument");
  ESP_REQUIRE(c->u, ESP_ERR_STATE, "ctx has no momentum buffer (cfg.momentum == 0)");
  ESP_REQUIRE(count == c->N * (size_t)c->w->nlocal, ESP_ERR_INVALID_ARG, "count must be nlocal * numel");
  ESP_CUDA(cudaSetDevice(c->w->dev));
  ESP_CUDA(cudaDeviceSynchronize());
  apply_zrec(c);
  ESP_CUDA(cudaMemcpy(host, c->u, 4 * count, cudaMemcpyDeviceToHost));
  ESP_API_END
}

esp_status_t esp_ctx_set_momentum(esp_ctx_t c, const float* host, size_t count) {
  ESP_API_BEGIN
  ESP_REQUIRE(c && host, ESP_ERR_INVALID_ARG, "null argument");
  ESP_REQUIRE(c->u, ESP_ERR_STATE, "ctx has no momentum buffer (cfg.momentum == 0)");
  ESP_REQUIRE(count == c->N * (size_t)c->w->nlocal, ESP_ERR_INVALID_ARG, "count must be nlocal * numel");
  ESP_CUDA(cudaSetDevice(c->w->dev));
  ESP_CUDA(cudaDeviceSynchronize());
  apply_zrec(c);   // r's pending zeros stay applied; u is overwritten below
  ESP_CUDA(cudaMemcpy(c->u, host, 4 * count, cudaMemcpyHostToDevice));
  ESP_API_END
}

esp_status_t esp_compress(esp_ctx_t c, const float* grad, void* payload, void* stream) {
  ESP_API_BEGIN
  ESP_REQUIRE(c, ESP_ERR_INVALID_ARG, "ctx is NULL");
  check_ptr16(grad, "grad");
  check_ptr16(payload, "payload");
  ESP_REQUIRE(c->cfg.kind != ESP_NONE, ESP_ERR_UNSUPPORTED, "NONE has no compressed payload");
  ESP_REQUIRE(c->w->hier_g == 0, ESP_ERR_UNSUPPORTED, "h1 of a hierarchical ctx: use its shard's world");
  ESP_CUDA(cudaSetDevice(c->w->dev));
  execute_compress(get_plan(c->w, {c}), grad, payload, as_stream(stream));
  ESP_API_END
}

esp_status_t esp_decompress(esp_ctx_t c, const void* const* pieces, int npieces, float* out_user, int accumulate,
                            void* stream) {
  ESP_API_BEGIN
  ESP_REQUIRE(accumulate == 0 || accumulate == 1, ESP_ERR_INVALID_ARG, "accumulate must be 0 or 1");
  ESP_REQUIRE(c && pieces && npieces >= 1 && npieces <= 64, ESP_ERR_INVALID_ARG, "bad argument");
  check_ptr16(out_user, "out");
  ESP_REQUIRE(c->cfg.kind != ESP_NONE, ESP_ERR_UNSUPPORTED, "NONE has no compressed payload");
  ESP_REQUIRE(c->w->hier_g == 0, ESP_ERR_UNSUPPORTED, "h2 of a hierarchical ctx: use its shard's world");
  for (int i = 0; i < npieces; ++i) check_ptr16(pieces[i], "piece");
  ESP_CUDA(cudaSetDevice(c->w->dev));
  cudaStream_t st = as_stream(stream);
  auto& D = c->dec;
  // accumulate: the aggregate goes to a per-ctx temporary, then out += it
  if (accumulate && !D.acc) ESP_CUDA(cudaMalloc(&D.acc, sizeof(float) * std::max<uint64_t>(c->N, 4)));
  float* out = accumulate ? D.acc : out_user;
  const bool tiles = c->cfg.kind == ESP_DGC || c->cfg.kind == ESP_TOPK;
  const bool hit = D.valid && D.out == out && D.pieces.size() == (size_t)npieces &&
                   std::equal(D.pieces.begin(), D.pieces.end(), pieces);
  auto stage = [&](size_t bytes) -> unsigned char* {   // pinned staging, reused once its last copy ran
    if (D.pending) ESP_CUDA(cudaEventSynchronize(D.ev));
    D.pending = false;
    if (bytes > D.hcap) {
      if (D.h) ESP_CUDA(cudaFreeHost(D.h));
      D.h = nullptr;
      ESP_CUDA(cudaMallocHost((void**)&D.h, bytes));
      D.hcap = bytes;
    }
    if (!D.ev) ESP_CUDA(cudaEventCreateWithFlags(&D.ev, cudaEventDisableTiming));
    return D.h;
  };
  auto copied = [&]() {
    ESP_CUDA(cudaEventRecord(D.ev, st));
    D.pending = true;
  };
  // dyn words: out pointer, step of the last compression (Randomk regenerates indices)
  const uint64_t step_now = c->step ? c->step - 1 : 0;
  if (!hit) {
    // tables for: one segment per partition, npieces pieces each
    std::vector<SegH2> segs;
    std::vector<uint32_t> units;
    std::vector<const unsigned char*> pp;
    std::vector<uint32_t> rt;
    std::vector<uint4> jobs;
    std::vector<size_t> toff_words;
    size_t toff_total = 0;
    const float divisor = c->cfg.reduce == ESP_MEAN ? (float)npieces : 1.0f;
    uint32_t u0 = 0;
    for (int p = 0; p < c->P; ++p) {
      const uint32_t len = c->phi[p] - c->plo[p];
      if (!len) continue;
      SegH2 s{};
      s.ooff = c->plo[p];
      s.hash = c->hash_base;
      s.part = (uint32_t)p;
      s.n = len;
      s.k = k_of(len, c->cfg.ratio);
      s.kpad = c->kpad;
      s.npieces = (uint32_t)npieces;
      s.piece0 = (uint32_t)pp.size();
      s.divisor = divisor;
      for (int i = 0; i < npieces; ++i) {
        pp.push_back((const unsigned char*)pieces[i] + (size_t)p * c->chunk_bytes);
        rt.push_back(c->cfg.randomk_shared_indices ? 0u : (uint32_t)i + 1);
      }
      s.nunits = div_up(len, tiles ? kTile : is_quant(c->cfg.kind) ? kSignUnit : kUnit);
      s.unit0 = u0;
      u0 += s.nunits;
      for (uint32_t i = 0; i < s.nunits; ++i) units.push_back((uint32_t)segs.size());
      if (tiles) {
        toff_words.push_back(toff_total);
        toff_total += (size_t)npieces * (s.nunits + 1);
        for (int i = 0; i < npieces; ++i)
          for (uint32_t e = 0; e < s.kpad; e += kOffJob) jobs.push_back(make_uint4((uint32_t)segs.size(), i, e, 0));
      }
      segs.push_back(s);
    }
    const size_t b_dyn = 16, b_seg = segs.size() * sizeof(SegH2), b_units = units.size() * 4;
    const size_t b_pp = pp.size() * 8, b_rt = rt.size() * 4, b_ps = jobs.size() * 16;
    D.off_seg = round_up(b_dyn, 256);
    D.off_units = round_up(D.off_seg + b_seg, 256);
    D.off_pp = round_up(D.off_units + b_units, 256);
    D.off_rt = round_up(D.off_pp + b_pp, 256);
    D.off_ps = round_up(D.off_rt + b_rt, 256);
    const size_t off_toff = round_up(D.off_ps + b_ps, 256);
    const size_t total = round_up(off_toff + toff_total * 4, 256);
    if (total > D.dcap) {   // grows rarely: the only synchronising step of a table change
      if (D.d) {
        ESP_CUDA(cudaStreamSynchronize(st));
        ESP_CUDA(cudaFree(D.d));
      }
      D.d = nullptr;
      ESP_CUDA(cudaMalloc((void**)&D.d, total));
      D.dcap = total;
    }
    unsigned char* d = D.d;
    for (size_t i = 0; i < segs.size(); ++i) {
      segs[i].optr = reinterpret_cast<const uint64_t*>(d);
      segs[i].step = reinterpret_cast<const uint64_t*>(d + 8);
      if (tiles) segs[i].toff = reinterpret_cast<uint32_t*>(d + off_toff) + toff_words[i];
    }
    unsigned char* h = stage(D.off_ps + b_ps);
    const uint64_t dyn[2] = {(uint64_t)(uintptr_t)out, step_now};
    std::memcpy(h, dyn, 16);
    std::memcpy(h + D.off_seg, segs.data(), b_seg);
    std::memcpy(h + D.off_units, units.data(), b_units);
    std::memcpy(h + D.off_pp, pp.data(), b_pp);
    std::memcpy(h + D.off_rt, rt.data(), b_rt);
    std::memcpy(h + D.off_ps, jobs.data(), b_ps);
    // (the toff region is written by h2_sparse_offsets every call)
    ESP_CUDA(cudaMemcpyAsync(d, h, D.off_ps + b_ps, cudaMemcpyHostToDevice, st));
    copied();
    D.pieces.assign(pieces, pieces + npieces);
    D.out = out;
    D.nunits = u0;
    D.njobs = (int)jobs.size();
    D.step_uploaded = step_now;
    D.valid = true;
  } else if (c->cfg.kind == ESP_RANDOMK && D.step_uploaded != step_now) {
    unsigned char* h = stage(16);
    const uint64_t dyn[2] = {(uint64_t)(uintptr_t)out, step_now};
    std::memcpy(h, dyn, 16);
    ESP_CUDA(cudaMemcpyAsync(D.d, h, 16, cudaMemcpyHostToDevice, st));
    copied();
    D.step_uploaded = step_now;
  }
  unsigned char* d = D.d;
  const size_t off_seg = D.off_seg, off_units = D.off_units, off_pp = D.off_pp, off_rt = D.off_rt,
               off_ps = D.off_ps;
  const uint32_t u0 = D.nunits;
  const int njobs = D.njobs;
  const SegH2* dseg = reinterpret_cast<const SegH2*>(d + off_seg);
  const uint32_t* dunits = reinterpret_cast<const uint32_t*>(d + off_units);
  const unsigned char* const* dpp = reinterpret_cast<const unsigned char* const*>(d + off_pp);
  const uint32_t* drt = reinterpret_cast<const uint32_t*>(d + off_rt);
  switch (c->cfg.kind) {
    case ESP_DGC: case ESP_TOPK:
      launch_h2_sparse(dseg, dunits, (int)u0, reinterpret_cast<const uint4*>(d + off_ps), njobs, dpp, npieces,
                       h2_sparse_dense((double)c->kpad * npieces, (double)c->N), st);
      break;
    case ESP_RANDOMK: launch_h2_randomk(dseg, dunits, (int)u0, dpp, drt, st); break;
    case ESP_EFSIGNSGD: launch_h2_sign(K_EFSIGN, dseg, dunits, (int)u0, dpp, npieces, st); break;
    default: launch_h2_sign(K_ONEBIT, dseg, dunits, (int)u0, dpp, npieces, st); break;
  }
  if (accumulate) launch_add(out_user, D.acc, (uint32_t)c->N, st);   // out = fl(out + aggregate)
  ESP_CUDA(cudaGetLastError());
  ESP_API_END
}

esp_status_t esp_sync_many(esp_world_t w, const esp_ctx_t* ctxs, float* const* grads, int ntensors,
                           void* stream) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && ctxs && grads && ntensors >= 1, ESP_ERR_INVALID_ARG, "bad argument");
  std::vector<esp_ctx_s*> v(ctxs, ctxs + ntensors);
  for (int i = 0; i < ntensors; ++i) check_ptr4(grads[i], "grad");
  ESP_REQUIRE(!w->loopback, ESP_ERR_STATE, "a loopback world syncs through esp_sync_many_loopback");
  // a cached plan was built from exactly this validated ctx list
  Plan* p = find_plan(w, v);
  if (!p) {
    std::set<esp_ctx_s*> seen;
    for (int i = 0; i < ntensors; ++i) {
      ESP_REQUIRE(v[i], ESP_ERR_INVALID_ARG, "ctx is NULL");
      ESP_REQUIRE(w->ctxs.count(v[i]) && v[i]->w == w, ESP_ERR_STATE, "ctx belongs to another world");
      ESP_REQUIRE(seen.insert(v[i]).second, ESP_ERR_INVALID_ARG, "ctx listed twice");
    }
  }
  ESP_CUDA(cudaSetDevice(w->dev));
  if (w->hier_g > 0) {
    execute_hier(w, v, grads, as_stream(stream));
    return ESP_OK;
  }
  if (!p) p = get_plan(w, v);
  execute_plan(p, grads, as_stream(stream));
  ESP_API_END
}

esp_status_t esp_sync_many_loopback(const esp_world_t* worlds, int nranks, const esp_ctx_t* ctxs,
                                    float* const* grads, int ntensors, void* stream) {
  ESP_API_BEGIN
  ESP_REQUIRE(worlds && ctxs && grads && nranks >= 2 && ntensors >= 1, ESP_ERR_INVALID_ARG, "bad argument");
  std::vector<Plan*> plans(nranks);
  std::vector<float* const*> gr(nranks);
  for (int r = 0; r < nranks; ++r) {
    esp_world_s* w = worlds[r];
    ESP_REQUIRE(w && w->loopback && w->nranks == nranks && w->rank == r, ESP_ERR_STATE,
                "worlds[r] must be rank r of one loopback group");
    ESP_REQUIRE(w->dev == worlds[0]->dev, ESP_ERR_STATE, "a loopback group lives on one device");
    std::vector<esp_ctx_s*> v(ctxs + (size_t)r * ntensors, ctxs + (size_t)(r + 1) * ntensors);
    for (int i = 0; i < ntensors; ++i) {
      ESP_REQUIRE(v[i] && v[i]->w == w, ESP_ERR_STATE, "ctxs[r][i] must belong to worlds[r]");
      check_ptr4(grads[(size_t)r * ntensors + i], "grad");
    }
    ESP_CUDA(cudaSetDevice(w->dev));
    gr[r] = grads + (size_t)r * ntensors;
    if (worlds[0]->hier_g > 0) continue;
    plans[r] = get_plan(w, v);
  }
  if (worlds[0]->hier_g > 0) {
    std::vector<esp_world_s*> ws(worlds, worlds + nranks);
    std::vector<std::vector<esp_ctx_s*>> cs(nranks);
    for (int r = 0; r < nranks; ++r) cs[r].assign(ctxs + (size_t)r * ntensors, ctxs + (size_t)(r + 1) * ntensors);
    execute_hier_loopback(ws, cs, gr, as_stream(stream));
    return ESP_OK;
  }
  execute_loopback(plans, gr, as_stream(stream));
  ESP_API_END
}

esp_status_t esp_sync(esp_world_t w, esp_ctx_t c, float* grad_inout, void* stream) {
  ESP_API_BEGIN
  ESP_REQUIRE(!w || !w->loopback, ESP_ERR_STATE, "a loopback world syncs through esp_sync_many_loopback");
  ESP_REQUIRE(w && c, ESP_ERR_INVALID_ARG, "null argument");
  ESP_REQUIRE(c->w == w, ESP_ERR_STATE, "ctx belongs to another world");
  check_ptr4(grad_inout, "grad");
  ESP_CUDA(cudaSetDevice(w->dev));
  if (w->hier_g > 0) {
    execute_hier(w, {c}, &grad_inout, as_stream(stream));
    return ESP_OK;
  }
  execute_plan(get_plan(w, {c}), &grad_inout, as_stream(stream));
  ESP_API_END
}

esp_status_t esp_last_timing(esp_world_t w, esp_timing_t* out) {
  ESP_API_BEGIN
  ESP_REQUIRE(w && out, ESP_ERR_INVALID_ARG, "null argument");
  *out = w->last;
  ESP_API_END
}

}  // extern "C"
