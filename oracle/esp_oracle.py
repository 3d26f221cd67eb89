"""ORACLE for the Espresso (arXiv 2205.14465) compressed gradient-sync hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` legs may import this module.
The product path (`paper_2205_14465_b200/`) never imports it and shares no code
with it: no kernels, headers, helpers, tables or constants.

A plain, slow, obviously-correct CPU implementation in numpy.  It simulates n
data-parallel ranks of one synchronisation of one tensor: every rank compresses
its gradient with error feedback (h1), the chosen collective routine moves the
payloads (with byte counters), and every rank decompresses and aggregates (h2).

Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
Readings of silent/garbled passages are numbered R1..R18 as in DESIGN.md
"Readings of the paper".

Pins (tests/test_oracle_*.py, marker "not gpu"):
  * top-k / DGC         brute force over itertools on tiny inputs, a heap-based
                        independent selection, tie-heavy bf16 inputs, special cases
  * sparse EF           exact invariant  transmitted + r_new == acc  (bit for bit)
  * sign EF             |delta + r_new - acc| <= 1/2 ulp(r_new); closed form scale
                        for all-equal magnitudes; fp64 / Fraction cross-check
  * Onebit              closed-form class means; same EF bound
  * Randomk             one index per stratum, ascending, distinct; chi-square
                        uniformity; determinism; shared across ranks.  Beyond these
                        invariants the sampler is DEFINED by this oracle (R5) —
                        "parity unpinned" for the exact index choice.
  * aggregation         rank-order fp32 sum vs fp64 mean within 1e-6 relative
  * routines            routine equivalences, n = 1, rho = 1 reductions
  * second residual r2  multi-step two-level EF telescoping for process 2 of both
                        divisible routines (sum out + r2_T + mean r_T == mean sum g);
                        exact closed-form a7 (scale2 = mean|A + r2|, class means)
                        with a non-zero r2 on an input where every step is exact
  * bytes on wire       closed forms of the cost table, S:131-150 numbers
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

# --------------------------------------------------------------------------
# vocabulary (P:1057-1070 routines table; P:1096-1114 action tasks)
# --------------------------------------------------------------------------
KINDS = ("none", "randomk", "dgc", "topk", "efsignsgd", "onebit")
ROUTINES = ("allreduce", "allgather", "alltoall_allgather", "gather_broadcast",
            "reducescatter_allgather", "reduce_broadcast")
SPARSE = ("randomk", "dgc", "topk")
QUANTIZED = ("efsignsgd", "onebit")
DIVISIBLE = ("alltoall_allgather", "gather_broadcast", "reducescatter_allgather", "reduce_broadcast")


@dataclass
class Cfg:
    kind: str
    ratio: float = 0.01
    error_feedback: bool = True
    seed: int = 0
    shared_indices: bool = True   # Randomk (R5)
    reduce: str = "mean"          # R9
    process: int = 0              # Alltoall/Allgather, Gather/Broadcast: 1 or 2 (0: the table's choice, R19)
    momentum: float = 0.0         # DGC momentum correction factor m (R20); 0 = plain error feedback
    approx: bool = False          # DGC approximate-count mode (R22): keep what passes the sampled threshold
    sample_rate: float = 0.0      # DGC sampler size (R22): 0 = 4096 samples, else about rate * N (<= 4096)


def process_of(cfg: Cfg) -> int:
    """The two processes of the divisible routines (App. A, P:66-87 and
    P:93-115): process 1 forwards the first compression's chunks (decompress n^2
    resp. n pieces); process 2 decompresses, aggregates and recompresses
    mid-scheme.  "We take the first process for sparse tensors and the second
    process for quantized tensors in Table ..., but the decision tree
    abstraction covers all of them": 0 selects that default."""
    if cfg.process in (1, 2):
        return cfg.process
    return 1 if cfg.kind in SPARSE else 2


def legal(cfg: Cfg, routine: str) -> bool:
    """Legal (compressor, routine) pairs.  UT row vs CT row of the routines table
    (P:1064-1065); "Compressed tensors cannot use Allreduce"; an
    allreducible compressed tensor may use Allreduce."""
    if cfg.kind == "none":
        return routine in ("allreduce", "reducescatter_allgather", "reduce_broadcast")
    if routine in ("allgather", "alltoall_allgather", "gather_broadcast"):
        return True
    return cfg.kind == "randomk" and cfg.shared_indices and routine == "allreduce"


# --------------------------------------------------------------------------
# sizes (R1, R10)
# --------------------------------------------------------------------------
def k_of(numel: int, ratio: float) -> int:
    """R1: k = min(N, max(1, ceil(rho*N))); 0 for an empty partition."""
    if numel == 0:
        return 0
    return min(numel, max(1, math.ceil(ratio * numel)))


def nparts_of(routine: str, n: int) -> int:
    """Divisible schemes partition the tensor into n parts; the first
    compression of Alltoall/Allgather is per partition (R10).  Gather/Broadcast
    compresses the whole tensor."""
    return n if routine == "alltoall_allgather" else 1


def partitions(numel: int, nparts: int):
    """R10: contiguous ranges of L = ceil(N/n) rounded up to a multiple of 32;
    the last non-empty partition takes the remainder, later ones may be empty."""
    if nparts == 1:
        return [(0, numel)]
    L = -(-numel // nparts)
    L = -(-L // 32) * 32
    return [(min(numel, p * L), min(numel, (p + 1) * L)) for p in range(nparts)]


def _r4(x):
    return -(-x // 4) * 4


def chunk_bytes(cfg: Cfg, numel: int, nparts: int) -> int:
    """Payload layout: every chunk of a tensor has
    the same size; sections are 16-byte aligned."""
    parts = partitions(numel, nparts)
    if cfg.kind in ("dgc", "topk"):
        kp = max(k_of(hi - lo, cfg.ratio) for lo, hi in parts)
        return 8 * _r4(kp)
    if cfg.kind == "randomk":
        kp = max(k_of(hi - lo, cfg.ratio) for lo, hi in parts)
        return 4 * _r4(kp)
    if cfg.kind in QUANTIZED:
        w = max(-(-(hi - lo) // 32) for lo, hi in parts)
        return 16 + 4 * _r4(w)
    if cfg.kind == "none":
        return 4 * numel
    raise ValueError(cfg.kind)


# --------------------------------------------------------------------------
# exact arithmetic helpers
# --------------------------------------------------------------------------
def key(x: np.ndarray) -> np.ndarray:
    """|x| as an order-preserving uint32: bits(x) & 0x7FFFFFFF (R2)."""
    return np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) & np.uint32(0x7FFFFFFF)


def exact_sum(x: np.ndarray) -> Fraction:
    """The exact real sum of an fp32 array, as a Fraction.  Each fp32 value is
    mant * 2^(e-150) (mant < 2^24); same-exponent mantissas are summed exactly
    in 12-bit halves with float64 bincounts (< 2^53), then combined as integers."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    if u.size == 0:
        return Fraction(0)
    e = ((u >> 23) & 0xFF).astype(np.int64)
    m = (u & 0x7FFFFF).astype(np.int64)
    m = np.where(e > 0, m | 0x800000, m)
    e = np.where(e > 0, e, 1)
    sgn = np.where((u >> 31) == 1, -1.0, 1.0)
    hi = np.bincount(e, weights=sgn * (m >> 12), minlength=256)
    lo = np.bincount(e, weights=sgn * (m & 0xFFF), minlength=256)
    total = 0
    for ee in range(1, 256):
        if hi[ee] or lo[ee]:
            total += ((int(hi[ee]) << 12) + int(lo[ee])) << (ee - 1)
    return Fraction(total, 1 << 149)


def f64(fr: Fraction) -> float:
    """Correctly rounded fp64 of an exact value."""
    return float(fr)


# --------------------------------------------------------------------------
# compressors on one segment (a whole tensor or one partition)
# --------------------------------------------------------------------------
def topk_select(acc: np.ndarray, k: int) -> np.ndarray:
    """Top-k by |x| (R2, R3).  Definition: stable-sort the indices by key
    descending (ties keep ascending index order), take the first k, and emit
    them sorted by index."""
    kk = key(acc).astype(np.int64)
    order = np.argsort(-kk, kind="stable")
    return np.sort(order[:k]).astype(np.uint32)


MASK64 = (1 << 64) - 1

# --------------------------------------------------------------------------
# DGC sampled threshold (reading R22; DGC is cited at P:828 and run at 1%,
# P:1426).  Only the approximate-count mode's RESULT depends on it; the exact
# mode uses it as an accelerator and the oracle does not compute it there.
# --------------------------------------------------------------------------
DGC_SAMPLE = 4096          # samples per segment: 512 strata x 8 consecutive elements
DGC_MARGIN = 4.0           # exact mode: j* = ceil(rho s + 4 sqrt(rho s)) (over-sampled)


def dgc_segment_hash(tensor_id: int, part: int, recompress: bool = False) -> int:
    """Per-segment sampler key (R22): splitmix64(tensor * 0x100000001b3 + part)
    for the first compression, + 0x9e37 for the mid-scheme recompression."""
    return splitmix64((tensor_id * 0x100000001B3 + (0x9E37 if recompress else 0) + part) & MASK64)


def dgc_strata(n: int, sample_rate: float) -> int:
    """R22: strata of 8 samples each: 512 by default (4096 samples), else
    ceil(rate * n / 8) clipped to [1, 512]."""
    if sample_rate <= 0.0:
        return DGC_SAMPLE // 8
    return max(1, min(DGC_SAMPLE // 8, math.ceil(sample_rate * n / 8)))


def dgc_sample_positions(n: int, seg_hash: int, strata: int = DGC_SAMPLE // 8) -> np.ndarray:
    """R22: for n > 4096, stratum G = [floor(G n / S), floor((G+1) n / S))
    (G < S strata) contributes the 8 consecutive elements starting at
    a_G + floor(u32(splitmix64(hash ^ G)) * (b_G - a_G - 7) / 2^32); for
    n <= 4096 the sample is the whole segment."""
    if n <= DGC_SAMPLE:
        return np.arange(n, dtype=np.int64)
    j = np.arange(8 * strata, dtype=np.uint64)
    G = j >> np.uint64(3)
    a = (G * np.uint64(n)) // np.uint64(strata)
    b = ((G + np.uint64(1)) * np.uint64(n)) // np.uint64(strata)
    h = splitmix64(np.uint64(seg_hash) ^ G) & np.uint64(0xFFFFFFFF)
    off = (h * (b - a - np.uint64(7))) >> np.uint64(32)
    return (a + off + (j & np.uint64(7))).astype(np.int64)


def dgc_threshold(acc: np.ndarray, k: int, ratio: float, seg_hash: int, approx: bool,
                  sample_rate: float = 0.0) -> int:
    """R22: the key threshold of the sampled-threshold selection: the need-th
    largest sampled key with its low 10 bits cleared (the 21-bit radix prefix
    the GPU selects in two histogram rounds).  need = k when the sample is the
    whole segment; else ceil(rho s + 4 sqrt(rho s)) (exact mode: enough that
    >= k pass w.h.p.) or max(1, round(rho s)) (approximate-count mode: about
    k pass in expectation); clipped to [1, s]."""
    n = acc.size
    pos = dgc_sample_positions(n, seg_hash, dgc_strata(n, sample_rate))
    sk = np.sort(key(acc)[pos])[::-1]
    s = sk.size
    if n <= DGC_SAMPLE:
        need = k
    else:
        rs = ratio * s
        need = int(math.floor(rs + 0.5)) if approx else int(math.ceil(rs + DGC_MARGIN * math.sqrt(rs)))
        need = max(1, min(s, need))
    return int(sk[need - 1]) & ~0x3FF


def dgc_approx_select(acc: np.ndarray, k: int, thr: int) -> np.ndarray:
    """Approximate-count DGC (R22, DGC's own selection): every element whose
    key passes the sampled threshold; when more than k pass, exactly the top-k
    of them (DGC's hierarchical re-selection) -- which is the segment's top-k.
    Emitted sorted by index."""
    passing = np.nonzero(key(acc) >= np.uint32(thr))[0]
    if passing.size <= k:
        return passing.astype(np.uint32)
    return topk_select(acc, k)


def splitmix64(z):
    """splitmix64 finaliser (Steele et al.), on Python ints or uint64 arrays."""
    if isinstance(z, np.ndarray):
        z = z.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def randomk_indices(seg_len: int, k: int, seed: int, tensor_id: int, step: int, part: int,
                    rank: int | None) -> np.ndarray:
    """R5: stratified hash sampler.  Stratum j = [floor(jN/k), floor((j+1)N/k));
    idx_j = start_j + H(j) mod len_j with H(j) = splitmix64(h ^ j) and
    h = splitmix64 chain over (seed, tensor, step, partition, rank+1 or 0 when
    shared).  Indices are relative to the segment start."""
    if k == 0:
        return np.zeros(0, np.uint32)
    h = splitmix64(seed & MASK64)
    for v in (tensor_id, step, part, 0 if rank is None else rank + 1):
        h = splitmix64(h ^ (v & MASK64))
    j = np.arange(k, dtype=np.uint64)
    n64 = np.uint64(seg_len)
    start = (j * n64) // np.uint64(k)
    end = ((j + np.uint64(1)) * n64) // np.uint64(k)
    hj = splitmix64(np.uint64(h) ^ j)
    return (start + hj % (end - start)).astype(np.uint32)


def l1_scale(p: np.ndarray) -> np.float32:
    """R7: EFSignSGD scale = ||p||_1 / N, computed as
    (float)((double)exact(sum|p|) / N)."""
    if p.size == 0:
        return np.float32(0.0)
    return np.float32(f64(exact_sum(np.abs(p))) / p.size)


def class_means(p: np.ndarray):
    """R8: Onebit reconstruction values: mean of {p >= 0} and mean of {p < 0}
    (0 when a class is empty), each (float)((double)exact(sum) / count)."""
    pos = p >= 0
    npos, nneg = int(pos.sum()), int((~pos).sum())
    mpos = np.float32(f64(exact_sum(p[pos])) / npos) if npos else np.float32(0.0)
    mneg = np.float32(f64(exact_sum(p[~pos])) / nneg) if nneg else np.float32(0.0)
    return mneg, mpos


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """bit l of word w <-> element 32w + l (LSB first); tail bits 0."""
    w = -(-bits.size // 32)
    b = np.zeros(w * 32, np.uint64)
    b[:bits.size] = bits
    shifts = np.arange(32, dtype=np.uint64)
    return (b.reshape(w, 32) << shifts).sum(axis=1).astype(np.uint32)


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    shifts = np.arange(32, dtype=np.uint32)
    b = (words.astype(np.uint32)[:, None] >> shifts) & np.uint32(1)
    return b.reshape(-1)[:n].astype(bool)


@dataclass
class Chunk:
    """A decoded view of one compressed chunk (one segment)."""
    kind: str
    seg_len: int
    idx: np.ndarray | None = None     # sparse: uint32 relative indices (sorted)
    val: np.ndarray | None = None     # sparse / randomk values
    words: np.ndarray | None = None   # quantized
    scale: np.float32 | None = None   # efsignsgd
    mneg: np.float32 | None = None    # onebit
    mpos: np.float32 | None = None


def compress_segment(cfg: Cfg, acc: np.ndarray, *, tensor_id=0, step=0, part=0, rank=0, recompress=False):
    """h1 on one segment.  Returns (chunk, transmitted) where `transmitted` is the
    dense fp32 vector the chunk decodes to (so that r_new = acc - transmitted for
    EF, G5 / P:1427: e <- (g+e) - C(g+e))."""
    n = acc.size
    if cfg.kind == "dgc" and cfg.approx:
        k = k_of(n, cfg.ratio)
        thr = (dgc_threshold(acc, k, cfg.ratio, dgc_segment_hash(tensor_id, part, recompress), True,
                             cfg.sample_rate) if n else 0)
        idx = dgc_approx_select(acc, k, thr)
        ch = Chunk(cfg.kind, n, idx=idx, val=acc[idx].copy())
    elif cfg.kind in ("dgc", "topk"):
        k = k_of(n, cfg.ratio)
        idx = topk_select(acc, k)
        ch = Chunk(cfg.kind, n, idx=idx, val=acc[idx].copy())
    elif cfg.kind == "randomk":
        k = k_of(n, cfg.ratio)
        idx = randomk_indices(n, k, cfg.seed, tensor_id, step, part,
                              None if cfg.shared_indices else rank)
        ch = Chunk(cfg.kind, n, idx=idx, val=acc[idx].copy())
    elif cfg.kind == "efsignsgd":
        ch = Chunk(cfg.kind, n, words=pack_bits(acc >= 0), scale=l1_scale(acc))
    elif cfg.kind == "onebit":
        mneg, mpos = class_means(acc)
        ch = Chunk(cfg.kind, n, words=pack_bits(acc >= 0), mneg=mneg, mpos=mpos)
    else:
        raise ValueError(cfg.kind)
    return ch, decompress_segment(ch)


def decompress_segment(ch: Chunk) -> np.ndarray:
    """h2 of one chunk: the dense vector it represents."""
    out = np.zeros(ch.seg_len, np.float32)
    if ch.kind in SPARSE:
        out[ch.idx.astype(np.int64)] = ch.val
    elif ch.kind == "efsignsgd":
        bits = unpack_bits(ch.words, ch.seg_len)
        out = np.where(bits, ch.scale, -ch.scale).astype(np.float32)
    elif ch.kind == "onebit":
        bits = unpack_bits(ch.words, ch.seg_len)
        out = np.where(bits, ch.mpos, ch.mneg).astype(np.float32)
    return out


def residual_update(acc: np.ndarray, transmitted: np.ndarray) -> np.ndarray:
    """Error feedback (G5): r_new = fl(acc - transmitted).  For sparse chunks the
    transmitted entries equal acc exactly, so r_new is acc with the selected
    entries set to 0 (the sparse EF invariant)."""
    return (acc - transmitted).astype(np.float32)


def serialize_chunk(cfg: Cfg, ch: Chunk, nbytes: int) -> bytes:
    """Byte layout of one chunk."""
    buf = bytearray(nbytes)
    if cfg.kind in ("dgc", "topk"):
        kp = nbytes // 8
        idx = np.full(kp, 0xFFFFFFFF, np.uint32)
        val = np.zeros(kp, np.float32)
        idx[:ch.idx.size] = ch.idx
        val[:ch.val.size] = ch.val
        buf[:4 * kp] = idx.tobytes()
        buf[4 * kp:] = val.tobytes()
    elif cfg.kind == "randomk":
        val = np.zeros(nbytes // 4, np.float32)
        val[:ch.val.size] = ch.val
        buf[:] = val.tobytes()
    elif cfg.kind == "efsignsgd":
        buf[0:4] = np.float32(ch.scale).tobytes()
        buf[16:16 + 4 * ch.words.size] = ch.words.astype("<u4").tobytes()
    elif cfg.kind == "onebit":
        buf[0:4] = np.float32(ch.mneg).tobytes()
        buf[4:8] = np.float32(ch.mpos).tobytes()
        buf[16:16 + 4 * ch.words.size] = ch.words.astype("<u4").tobytes()
    return bytes(buf)


# --------------------------------------------------------------------------
# aggregation (R9): fp32 sum in rank order starting from +0.0f, then / n
# --------------------------------------------------------------------------
def aggregate(dense_list, reduce: str, n: int) -> np.ndarray:
    acc = np.zeros(dense_list[0].size, np.float32)
    for d in dense_list:
        acc = (acc + d).astype(np.float32)
    if reduce == "mean":
        acc = (acc / np.float32(n)).astype(np.float32)
    return acc


# --------------------------------------------------------------------------
# per-rank state and counters
# --------------------------------------------------------------------------
@dataclass
class RankState:
    r: np.ndarray                      # EF residual (N); with momentum correction: v (R20)
    r2: np.ndarray | None = None       # second residual of a mid-scheme recompression (R11)
    step: int = 0
    u: np.ndarray | None = None        # DGC momentum buffer (R20)


def new_states(n: int, numel: int, routine: str, cfg: Cfg):
    st = []
    for rank in range(n):
        r2 = None
        p2 = cfg.kind != "none" and process_of(cfg) == 2
        if p2 and routine == "alltoall_allgather":
            lo, hi = partitions(numel, n)[rank]
            r2 = np.zeros(hi - lo, np.float32)
        elif p2 and routine == "gather_broadcast" and rank == 0:
            r2 = np.zeros(numel, np.float32)
        u = np.zeros(numel, np.float32) if cfg.momentum else None
        st.append(RankState(np.zeros(numel, np.float32), r2, u=u))
    return st


@dataclass
class Counters:
    h1: int = 0           # compress applications (h1(M) and h1(alpha M) each count 1)
    h2: int = 0           # decompressed pieces
    sent: int = 0
    recv: int = 0
    phases: list = field(default_factory=list)

    def comm(self, name, sent, recv):
        self.sent += sent
        self.recv += recv
        self.phases.append((name, sent, recv))


# --------------------------------------------------------------------------
# one synchronisation of one tensor across n simulated ranks
# --------------------------------------------------------------------------
@dataclass
class SyncResult:
    outs: list          # per rank aggregated tensor
    payloads: list      # per rank serialized first-compression payload (P chunks)
    payloads2: list     # per rank serialized mid-scheme payload (quantized P2) or None
    counters: list      # per rank Counters


def _compress_rank(cfg, routine, g, st, tensor_id, rank, n):
    """h1 with EF on one rank: acc = g + r; per-partition compression; r update.

    Momentum correction (DGC, R20): u = fl(fl(m u) + g) replaces g, the
    residual r plays DGC's accumulator v (acc = fl(u + v)), and after the
    selection both v and u are zeroed at the selected indices ("momentum factor
    masking")."""
    if cfg.momentum:
        if cfg.kind not in ("dgc", "topk") or not cfg.error_feedback:
            raise ValueError("momentum correction needs DGC/TOPK with error feedback")
        mu = (np.float32(cfg.momentum) * st.u).astype(np.float32)
        st.u = (mu + g.astype(np.float32)).astype(np.float32)
        g = st.u
    acc = (g + st.r).astype(np.float32) if cfg.error_feedback else g.astype(np.float32)
    P = nparts_of(routine, n)
    chunks, trans = [], np.zeros_like(acc)
    for p, (lo, hi) in enumerate(partitions(acc.size, P)):
        ch, t = compress_segment(cfg, acc[lo:hi], tensor_id=tensor_id, step=st.step, part=p, rank=rank)
        chunks.append(ch)
        trans[lo:hi] = t
        if cfg.momentum:
            st.u[lo + ch.idx.astype(np.int64)] = 0.0
    if cfg.error_feedback:
        st.r = residual_update(acc, trans)
    return chunks


def sync(routine: str, cfg: Cfg, grads, states, tensor_id: int = 0) -> SyncResult:
    """Run h1 -> routine -> h2 on n = len(grads) ranks (SURVEY.md 8c, App. A
    P:52-117).  `states` is updated in place (EF residuals, step counter)."""
    n = len(grads)
    N = grads[0].size
    if not legal(cfg, routine):
        raise ValueError(f"illegal pair {cfg.kind}/{routine}")
    cnt = [Counters() for _ in range(n)]
    if cfg.kind == "none":
        out = _sync_uncompressed(routine, cfg, grads, cnt)
        for st in states:
            st.step += 1
        return SyncResult([out.copy() for _ in range(n)], [None] * n, [None] * n, cnt)

    P = nparts_of(routine, n)
    cb = chunk_bytes(cfg, N, P)
    M = cb * P
    chunks = []
    for rank in range(n):
        chunks.append(_compress_rank(cfg, routine, grads[rank], states[rank], tensor_id, rank, n))
        cnt[rank].h1 += 1
    payloads = [b"".join(serialize_chunk(cfg, ch, cb) for ch in chunks[r]) for r in range(n)]
    payloads2 = [None] * n
    parts = partitions(N, P)

    if routine == "allreduce":
        # Randomk with shared indices: the value vectors are allreducible.
        for r in range(n):
            cnt[r].comm("allreduce", 2 * (n - 1) * M // n, 2 * (n - 1) * M // n)
        vals = aggregate([chunks[r][0].val for r in range(n)], cfg.reduce, n)
        ch = Chunk("randomk", N, idx=chunks[0][0].idx, val=vals)
        out = decompress_segment(ch)
        for r in range(n):
            cnt[r].h2 += 1
        outs = [out.copy() for _ in range(n)]

    elif routine == "allgather":
        for r in range(n):
            cnt[r].comm("allgather", (n - 1) * M, (n - 1) * M)
        out = aggregate([decompress_segment(chunks[r][0]) for r in range(n)], cfg.reduce, n)
        for r in range(n):
            cnt[r].h2 += n
        outs = [out.copy() for _ in range(n)]

    elif routine == "alltoall_allgather" and process_of(cfg) == 1:
        # process 1: Alltoall chunks (r -> j), Allgather the n received
        # chunks, decompress all n^2 pieces.
        for r in range(n):
            cnt[r].comm("alltoall", (n - 1) * cb, (n - 1) * cb)
            cnt[r].comm("allgather", (n - 1) * M, (n - 1) * M)
        out = np.zeros(N, np.float32)
        for p, (lo, hi) in enumerate(parts):
            out[lo:hi] = aggregate([decompress_segment(chunks[r][p]) for r in range(n)], cfg.reduce, n)
        for r in range(n):
            cnt[r].h2 += n * n
        outs = [out.copy() for _ in range(n)]

    elif routine == "alltoall_allgather":
        # process 2: rank j decompresses the n chunks of partition j,
        # aggregates, adds its second residual, recompresses (alpha = 1/n: the
        # same compressor on the partition, k_j = k_of(len_j) for sparse ones),
        # Allgather; everyone decompresses the n partitions.
        c2 = []
        for j in range(n):
            lo, hi = parts[j]
            A = aggregate([decompress_segment(chunks[r][j]) for r in range(n)], cfg.reduce, n)
            cnt[j].comm("alltoall", (n - 1) * cb, (n - 1) * cb)
            cnt[j].h2 += n
            st = states[j]
            q = (A + st.r2).astype(np.float32) if cfg.error_feedback else A
            ch, t = compress_segment(cfg, q, tensor_id=tensor_id, step=st.step, part=j, rank=j, recompress=True)
            if cfg.error_feedback:
                st.r2 = residual_update(q, t)
            cnt[j].h1 += 1
            c2.append(ch)
        for j in range(n):
            payloads2[j] = serialize_chunk(cfg, c2[j], cb)
            cnt[j].comm("allgather", (n - 1) * cb, (n - 1) * cb)
        out = np.zeros(N, np.float32)
        for p, (lo, hi) in enumerate(parts):
            out[lo:hi] = decompress_segment(c2[p])
        for r in range(n):
            cnt[r].h2 += n
        outs = [out.copy() for _ in range(n)]

    elif routine == "gather_broadcast" and process_of(cfg) == 1:
        # process 1: Gather to root 0 (R17), Broadcast all n payloads.
        cnt[0].comm("gather", 0, (n - 1) * M)
        for r in range(1, n):
            cnt[r].comm("gather", M, 0)
            cnt[r].comm("broadcast", 0, n * M)
        cnt[0].comm("broadcast", n * M if n > 1 else 0, 0)
        out = aggregate([decompress_segment(chunks[r][0]) for r in range(n)], cfg.reduce, n)
        for r in range(n):
            cnt[r].h2 += n
        outs = [out.copy() for _ in range(n)]

    elif routine == "gather_broadcast":
        # process 2 (R12, R14): root decompresses n payloads,
        # aggregates, adds r2, recompresses (alpha = 1), broadcasts one payload.
        cnt[0].comm("gather", 0, (n - 1) * M)
        for r in range(1, n):
            cnt[r].comm("gather", M, 0)
        A = aggregate([decompress_segment(chunks[r][0]) for r in range(n)], cfg.reduce, n)
        cnt[0].h2 += n
        st = states[0]
        q = (A + st.r2).astype(np.float32) if cfg.error_feedback else A
        ch, t = compress_segment(cfg, q, tensor_id=tensor_id, step=st.step, part=0, rank=0, recompress=True)
        if cfg.error_feedback:
            st.r2 = residual_update(q, t)
        cnt[0].h1 += 1
        payloads2[0] = serialize_chunk(cfg, ch, cb)
        cnt[0].comm("broadcast", M if n > 1 else 0, 0)
        for r in range(1, n):
            cnt[r].comm("broadcast", 0, M)
        out = decompress_segment(ch)
        for r in range(n):
            cnt[r].h2 += 1
        outs = [out.copy() for _ in range(n)]
    else:
        raise ValueError(routine)

    for st in states:
        st.step += 1
    return SyncResult(outs, payloads, payloads2, cnt)


def _sync_uncompressed(routine, cfg, grads, cnt):
    """UT routines: all three compute the mean (sum) of the raw
    gradients; they differ only in traffic.  Overall compression time 0."""
    n = len(grads)
    M = 4 * grads[0].size
    for r in range(n):
        if routine == "allreduce":
            cnt[r].comm("allreduce", 2 * (n - 1) * M // n, 2 * (n - 1) * M // n)
        elif routine == "reducescatter_allgather":
            cnt[r].comm("reducescatter", (n - 1) * M // n, (n - 1) * M // n)
            cnt[r].comm("allgather", (n - 1) * M // n, (n - 1) * M // n)
        elif routine == "reduce_broadcast":
            if r == 0:
                cnt[r].comm("reduce", 0, (n - 1) * M)
                cnt[r].comm("broadcast", M if n > 1 else 0, 0)
            else:
                cnt[r].comm("reduce", M, 0)
                cnt[r].comm("broadcast", 0, M)
    return aggregate([g.astype(np.float32) for g in grads], cfg.reduce, n)


# --------------------------------------------------------------------------
# cost table — closed forms; used as the bytes-on-wire oracle
# --------------------------------------------------------------------------
def table_comm_bytes(row: str, M: float, n: int) -> float:
    """Communication volume per rank in units of bytes (time * B) per row of the
    cost table, P:38-43 (R13: quantized Alltoall/Allgather uses the table's
    2(n-1)M/n)."""
    if n == 1:
        return 0.0
    return {
        "allreduce": 2 * (n - 1) * M / n,
        "allgather": (n - 1) * M,
        "alltoall_allgather_sparse": (n * n - 1) * M / n,
        "alltoall_allgather_quantized": 2 * (n - 1) * M / n,
        "gather_broadcast_sparse": (2 * n - 1) * M,
        "gather_broadcast_quantized": n * M,
    }[row]


def table_comm_time(row: str, M: float, n: int, B: float) -> float:
    return table_comm_bytes(row, M, n) / B


def table_compression_time(row: str, M: float, n: int, h1, h2) -> float:
    """Overall compression time column of P:38-43 (R12: Gather/Broadcast
    quantized decompresses full-size payloads, h2(M))."""
    return {
        "allreduce": h1(M) + h2(M),
        "allgather": h1(M) + n * h2(M),
        "alltoall_allgather_sparse": h1(M) + n * n * h2(M / n),
        "alltoall_allgather_quantized": h1(M) + h1(M / n) + 2 * n * h2(M / n),
        "gather_broadcast_sparse": h1(M) + n * h2(M),
        "gather_broadcast_quantized": 2 * h1(M) + (n + 1) * h2(M),
    }[row]


def table_row(cfg: Cfg, routine: str) -> str:
    if routine == "allreduce":
        return "allreduce"
    if routine == "allgather":
        return "allgather"
    # the table's "sparse" / "quantized" rows are processes 1 / 2
    t = "sparse" if process_of(cfg) == 1 else "quantized"
    return f"{routine}_{t}"


def table_ops(row: str, n: int):
    """(h1 applications, h2 applications) on the critical rank."""
    return {
        "allreduce": (1, 1),
        "allgather": (1, n),
        "alltoall_allgather_sparse": (1, n * n),
        "alltoall_allgather_quantized": (2, 2 * n),
        "gather_broadcast_sparse": (1, n),
        "gather_broadcast_quantized": (2, n + 1),
    }[row]


# --------------------------------------------------------------------------
# strategy selection (App. A; Algorithm 1
# P:1299-1361; readings R15, R21) -- test infrastructure like the rest
# --------------------------------------------------------------------------
def curve_eval(samples, nbytes: float) -> float:
    """Measured cost curve (input bytes, seconds), fitted log-log piecewise
    linearly ("curve fitting"); clamped below the first sample, the last
    segment extended above the last."""
    xs = [math.log(b) for b, _ in samples]
    ys = [math.log(t) for _, t in samples]
    if len(samples) == 1 or nbytes <= samples[0][0]:
        return samples[0][1]
    x = math.log(nbytes)
    i = 1
    while i < len(xs) - 1 and nbytes > samples[i][0]:
        i += 1
    return math.exp(ys[i - 1] + (ys[i] - ys[i - 1]) * (x - xs[i - 1]) / (xs[i] - xs[i - 1]))


def option_time(cfg: Cfg, routine: str, numel: int, n: int, B: float, h1, h2) -> float:
    """Predicted sync time of one tensor: the cost table's row for the option
     with M = its payload, h(.) keyed by input bytes (R15)."""
    if cfg.kind == "none":
        # the uncompressed routines' volumes: Allreduce 2(n-1)M/n;
        # Reduce-scatter (n-1)M/n + Allgather of the M/n shards (n-1)M/n;
        # Reduce (n-1)M + Broadcast of the M-byte result M
        M = 4.0 * numel
        if n == 1:
            return 0.0
        if routine == "allreduce":
            v = 2 * (n - 1) * M / n
        elif routine == "reducescatter_allgather":
            v = (n - 1) * M / n + (n - 1) * (M / n)
        else:
            v = (n - 1) * M + M
        return v / B
    P = nparts_of(routine, n)
    M = chunk_bytes(cfg, numel, P) * P
    row = table_row(cfg, routine)
    inb = 4.0 * numel
    f1 = lambda m: curve_eval(h1, inb if m == M else inb / n)   # h1(M) / h1(M/n)
    f2 = lambda m: curve_eval(h2, inb if m == M else inb / n)
    return table_comm_bytes(row, M, n) / B + table_compression_time(row, M, n, f1, f2)


def select_option(options, numel: int, n: int, B: float):
    """GetBestOption (Algorithm 1) for one tensor with no
    computation to overlap (R21): the fastest candidate, ties to the first."""
    best, bt = -1, 0.0
    for i, (cfg, routine, h1, h2) in enumerate(options):
        t = option_time(cfg, routine, numel, n, B, h1, h2)
        if best < 0 or t < bt:
            best, bt = i, t
    return best, bt


# --------------------------------------------------------------------------
# hierarchical communication (P:722-728 three phases,
# P:1085-1091 "only considers division schemes for intra-machine
# communications in hierarchical communication"; reading R23): n = m machines
# x g GPUs, rank r = machine r // g, local index r % g
# --------------------------------------------------------------------------
def hier_shard_tensor_id(tensor_id: int, shard: int) -> int:
    """R23: the inter-machine sync of shard i is its own tensor for the
    compressors' counter-based draws: id = tensor_id * 4096 + i."""
    return tensor_id * 4096 + shard


def new_states_hier(n: int, numel: int, routine: str, cfg: Cfg, g: int):
    """Rank (a, i) keeps the EF state of shard i as rank a of the m-rank
    inter-machine sync of that shard."""
    m = n // g
    shards = partitions(numel, g)
    return [new_states(m, shards[r % g][1] - shards[r % g][0], routine, cfg)[r // g] for r in range(n)]


def sync_hierarchical(routine: str, cfg: Cfg, grads, states, g: int, tensor_id: int = 0) -> SyncResult:
    """Three phases: (1) intra-machine Reduce-scatter of the
    uncompressed tensor -- shard i (R10 partitions into g parts) of machine a
    = rank-order fp32 mean over its g GPUs (SUM: the sum); (2) inter-machine:
    the m GPUs holding shard i run the compressed routine on it (any process;
    compression, EF and aggregation as in sync(), mean over the m machines);
    (3) intra-machine Allgather of the g shards.  The result is the mean of
    the machines' means."""
    n = len(grads)
    if g < 1 or n % g:
        raise ValueError("g must divide n")
    m = n // g
    N = grads[0].size
    if cfg.kind == "none" or not legal(cfg, routine) or routine not in ("allgather", "alltoall_allgather",
                                                                          "gather_broadcast"):
        raise ValueError(f"hierarchical sync of {cfg.kind}/{routine}")
    shards = partitions(N, g)
    cnt = [Counters() for _ in range(n)]
    # (1) intra-machine reduce-scatter (uncompressed): 4 (g-1)/g N bytes per rank
    mid = {}
    for a in range(m):
        for i, (lo, hi) in enumerate(shards):
            mid[a, i] = aggregate([grads[a * g + j][lo:hi].astype(np.float32) for j in range(g)], cfg.reduce, g) \
                if hi > lo else np.zeros(0, np.float32)
    for r in range(n):
        rs = sum(4 * (hi - lo) for j, (lo, hi) in enumerate(shards) if j != r % g)
        cnt[r].comm("intra_reducescatter", rs, 4 * (shards[r % g][1] - shards[r % g][0]) * (g - 1))
    # (2) inter-machine compressed sync of each shard
    final = {}
    for i, (lo, hi) in enumerate(shards):
        if hi == lo:
            for a in range(m):
                final[a, i] = np.zeros(0, np.float32)
            continue
        res = sync(routine, cfg, [mid[a, i] for a in range(m)], [states[a * g + i] for a in range(m)],
                   tensor_id=hier_shard_tensor_id(tensor_id, i))
        for a in range(m):
            final[a, i] = res.outs[a]
            c = res.counters[a]
            r = a * g + i
            cnt[r].h1 += c.h1
            cnt[r].h2 += c.h2
            cnt[r].comm("inter_" + routine, c.sent, c.recv)
    # (3) intra-machine allgather of the shards
    outs = []
    for r in range(n):
        a, i = divmod(r, g)
        out = np.zeros(N, np.float32)
        for j, (lo, hi) in enumerate(shards):
            out[lo:hi] = final[a, j]
        outs.append(out)
        mine = 4 * (shards[i][1] - shards[i][0])
        cnt[r].comm("intra_allgather", mine * (g - 1), sum(4 * (hi - lo) for j, (lo, hi) in enumerate(shards) if j != i))
    return SyncResult(outs, [None] * n, [None] * n, cnt)
