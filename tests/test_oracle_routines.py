"""Pins of the oracle's routine simulation: cost-table closed forms,
SPEC worked examples, special cases (n = 1, rho = 1), routine
equivalences and fp64 tolerance of the rank-order aggregation (no GPU)."""
import math

import numpy as np
import pytest

from oracle import esp_oracle as O
from synth.values import gradient

PAIRS = [(k, r) for k in O.KINDS for r in O.ROUTINES
         if O.legal(O.Cfg(k), r)]


def _grads(n, N, dist="D1", step=0):
    return [gradient(N, rank=r, step=step, dist=dist) for r in range(n)]


def test_legal_pairs_table():
    # UT routines only for uncompressed; CT routines for compressed;
    # compressed tensors cannot use Allreduce unless allreducible
    assert O.legal(O.Cfg("none"), "allreduce")
    assert not O.legal(O.Cfg("none"), "allgather")
    assert not O.legal(O.Cfg("dgc"), "allreduce")
    assert O.legal(O.Cfg("randomk", shared_indices=True), "allreduce")
    assert not O.legal(O.Cfg("randomk", shared_indices=False), "allreduce")
    assert not O.legal(O.Cfg("efsignsgd"), "reducescatter_allgather")
    assert len(PAIRS) == 3 + 4 * 3 + 4


@pytest.mark.parametrize("kind,routine", PAIRS)
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_bytes_on_wire_closed_forms(kind, routine, n):
    """Per-rank traffic of each phase, summed along the critical path, equals the
    cost table's communication volume."""
    cfg = O.Cfg(kind, 0.01)
    N = 4133
    res = O.sync(routine, cfg, _grads(n, N), O.new_states(n, N, routine, cfg))
    c = res.counters
    if kind == "none":
        M = 4 * N
        if routine == "allreduce":
            assert c[0].recv == pytest.approx(2 * (n - 1) * M / n, abs=n)
        elif routine == "reducescatter_allgather":
            assert c[1].recv == pytest.approx(2 * (n - 1) * M / n, abs=n)  # == Allreduce
        else:
            assert c[0].recv + c[1].recv == n * M           # (n-1)M reduce + M broadcast
        return
    P = O.nparts_of(routine, n)
    M = O.chunk_bytes(cfg, N, P) * P
    row = O.table_row(cfg, routine)
    if routine == "gather_broadcast":
        # critical path: root's gather receive + a non-root's broadcast receive
        got = c[0].phases[0][2] + c[1].phases[-1][2]
    else:
        got = c[1].recv
    # ring chunking rounds M/n down when n does not divide M
    assert got == pytest.approx(O.table_comm_bytes(row, M, n), rel=0, abs=n)
    # op counts of the table's compression column on the critical (root) rank
    assert (c[0].h1, c[0].h2) == O.table_ops(row, n)


def test_spec_cost_examples():
    # S:131-133, S:139-141 (B = 1.25e10 B/s, M = 1e8 B, n = 4)
    B, M = 1.25e10, 1e8
    assert O.table_comm_time("allreduce", M, 4, B) == pytest.approx(12e-3)
    assert O.table_comm_time("allgather", M, 4, B) == pytest.approx(24e-3)
    assert O.table_comm_time("alltoall_allgather_sparse", M, 4, B) == pytest.approx(30e-3)
    assert O.table_comm_time("gather_broadcast_quantized", M, 4, B) == pytest.approx(32e-3)
    assert O.table_comm_time("allreduce", 1e7, 2, 1e9) == pytest.approx(10e-3)
    for row in ("allreduce", "allgather", "alltoall_allgather_sparse",
                "alltoall_allgather_quantized", "gather_broadcast_sparse",
                "gather_broadcast_quantized"):
        assert O.table_comm_time(row, M, 1, B) == 0
    one = lambda m: 1e-3
    # S:147-150 constant curves h1 = h2 = 1 ms, n = 4
    assert O.table_compression_time("allgather", M, 4, one, one) == pytest.approx(5e-3)
    assert O.table_compression_time("alltoall_allgather_quantized", M, 4, one, one) == pytest.approx(10e-3)
    assert O.table_compression_time("allreduce", M, 4, one, one) == pytest.approx(2e-3)


def test_allreduce_equals_rs_ag_closed_form():
    # Allreduce = Reduce-scatter + Allgather, both 2(n-1)M/(nB)
    for n in (2, 4, 8):
        M = 2 ** 20
        rs = (n - 1) * M / n
        ag = (n - 1) * (M / n)
        assert rs + ag == pytest.approx(O.table_comm_bytes("allreduce", M, n))


@pytest.mark.parametrize("kind,routine", PAIRS)
def test_n1_is_decompress_of_compress(kind, routine):
    cfg = O.Cfg(kind, 0.05)
    g = gradient(1000)
    res = O.sync(routine, cfg, [g], O.new_states(1, 1000, routine, cfg))
    if kind == "none":
        assert np.array_equal(res.outs[0], g)
        return
    ch, t = O.compress_segment(cfg, g)
    assert np.array_equal(res.outs[0], t)


@pytest.mark.parametrize("kind", ["dgc", "topk", "randomk"])
@pytest.mark.parametrize("routine", ["allgather", "alltoall_allgather", "gather_broadcast"])
def test_rho1_reduces_to_uncompressed_mean(kind, routine):
    n, N = 4, 777
    cfg = O.Cfg(kind, 1.0)
    grads = _grads(n, N)
    st = O.new_states(n, N, routine, cfg)
    res = O.sync(routine, cfg, grads, st)
    ref = O.sync("allreduce", O.Cfg("none"), grads, O.new_states(n, N, "allreduce", O.Cfg("none")))
    assert np.array_equal(res.outs[0], ref.outs[0])
    assert all(np.all(s.r == 0) for s in st)


@pytest.mark.parametrize("kind", ["dgc", "topk", "randomk", "efsignsgd", "onebit"])
def test_sparse_gather_broadcast_equals_allgather(kind):
    n, N = 4, 3000
    cfg = O.Cfg(kind, 0.02)
    a = O.sync("allgather", cfg, _grads(n, N), O.new_states(n, N, "allgather", cfg))
    if kind in O.SPARSE:
        b = O.sync("gather_broadcast", cfg, _grads(n, N), O.new_states(n, N, "gather_broadcast", cfg))
        assert np.array_equal(a.outs[0], b.outs[0])
    for r in range(n):
        assert np.array_equal(a.outs[r], a.outs[0])


def test_aggregation_fp64_tolerance():
    """rank-order fp32 mean vs exact mean: within 1e-6 * mean|x| + denormal floor."""
    for n in (2, 4, 8):
        xs = _grads(n, 10000, dist="D2")
        got = O.aggregate(xs, "mean", n).astype(np.float64)
        ref = sum(x.astype(np.float64) for x in xs) / n
        scale = sum(np.abs(x.astype(np.float64)) for x in xs) / n
        assert np.all(np.abs(got - ref) <= 1e-6 * scale + 1e-38)
        s = O.aggregate(xs, "sum", n).astype(np.float64)
        assert np.all(np.abs(s - ref * n) <= 1e-6 * scale * n + 1e-38)


@pytest.mark.parametrize("kind", ["efsignsgd", "onebit"])
def test_quantized_alltoall_mid_scheme(kind):
    """Process 2: the output on partition j is the recompression of
    (mean of decompressed chunks + r2_j); r2 obeys the EF bound."""
    n, N = 4, 2000
    cfg = O.Cfg(kind)
    grads = _grads(n, N)
    st = O.new_states(n, N, "alltoall_allgather", cfg)
    res = O.sync("alltoall_allgather", cfg, grads, st)
    parts = O.partitions(N, n)
    for j, (lo, hi) in enumerate(parts):
        seg = res.outs[0][lo:hi]
        if kind == "efsignsgd":
            # decoded partition is +-scale2 with a single magnitude
            assert np.unique(np.abs(seg)).size <= 1
        else:
            assert np.unique(seg).size <= 2
    for r in range(n):
        assert np.array_equal(res.outs[r], res.outs[0])


def test_multistep_ef_telescopes():
    """sum_t transmitted_t + r_T == sum_t g_t (within fp32 rounding of T adds)."""
    N, T = 5000, 5
    for kind in ("dgc", "randomk", "efsignsgd", "onebit"):
        cfg = O.Cfg(kind, 0.01)
        st = O.new_states(1, N, "allgather", cfg)
        sum_t = np.zeros(N)
        sum_g = np.zeros(N)
        for t in range(T):
            g = gradient(N, step=t)
            res = O.sync("allgather", cfg, [g], st)
            sum_t += res.outs[0].astype(np.float64)
            sum_g += g.astype(np.float64)
        lhs = sum_t + st[0].r.astype(np.float64)
        tol = T * 2 * np.spacing(np.float32(np.abs(sum_g).max() + np.abs(sum_t).max())).astype(np.float64)
        assert np.max(np.abs(lhs - sum_g)) <= tol


def test_golden_cost_examples():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cost_examples.json")))
    for e in g["comm_time_s"]:
        assert O.table_comm_time(e["row"], e["M"], e["n"], e["B"]) == pytest.approx(e["t"]), e["cite"]
    one = lambda m: 1e-3
    for e in g["compression_time_const_1ms"]:
        assert O.table_compression_time(e["row"], 1e8, e["n"], one, one) == pytest.approx(e["t"]), e["cite"]
    for e in g["sparse_bytes"]:
        assert O.chunk_bytes(O.Cfg("dgc", e["ratio"]), e["numel"], 1) == e["bytes"]
    for e in g["one_bit_word_bytes"]:
        assert O.chunk_bytes(O.Cfg("efsignsgd"), e["numel"], 1) - 16 == e["bytes"]


# ---- the other process of each divisible routine ("the decision
# tree abstraction covers all of them"; reading R19) -------------------------
XPROC = [(k, r, p) for k in ("dgc", "topk", "randomk", "efsignsgd", "onebit")
         for r in ("alltoall_allgather", "gather_broadcast") for p in (1, 2)]


@pytest.mark.parametrize("kind,routine,process", XPROC)
@pytest.mark.parametrize("n", [2, 3, 4])
def test_process_bytes_and_ops_closed_forms(kind, routine, process, n):
    """Both processes of both divisible routines, for every compressor, move
    the bytes and apply the h1/h2 counts of the cost table's row for that
    process (rows "sparse" = process 1, "quantized" = process 2)."""
    cfg = O.Cfg(kind, 0.01, process=process)
    N = 4133
    res = O.sync(routine, cfg, _grads(n, N), O.new_states(n, N, routine, cfg))
    c = res.counters
    P = O.nparts_of(routine, n)
    M = O.chunk_bytes(cfg, N, P) * P
    row = O.table_row(cfg, routine)
    assert row.endswith("_sparse" if process == 1 else "_quantized")
    got = c[0].phases[0][2] + c[1].phases[-1][2] if routine == "gather_broadcast" else c[1].recv
    assert got == pytest.approx(O.table_comm_bytes(row, M, n), rel=0, abs=n)
    assert (c[0].h1, c[0].h2) == O.table_ops(row, n)
    for r in range(n):
        assert np.array_equal(res.outs[r], res.outs[0])


@pytest.mark.parametrize("kind", ["efsignsgd", "onebit", "dgc", "randomk"])
def test_process1_alltoall_equals_per_partition_allgather(kind):
    """Process 1 only forwards the first compression's chunks: its output is the
    rank-order mean of every rank's per-partition decompression -- which is
    exactly the process-1 Gather/Broadcast of per-partition payloads, and for a
    single partition (n = 1) decompress(compress(g))."""
    n, N = 4, 3001
    cfg = O.Cfg(kind, 0.02, process=1)
    grads = _grads(n, N)
    res = O.sync("alltoall_allgather", cfg, grads, O.new_states(n, N, "alltoall_allgather", cfg))
    parts = O.partitions(N, n)
    ref = np.zeros(N, np.float32)
    for p, (lo, hi) in enumerate(parts):
        dec = []
        for r in range(n):
            acc = grads[r][lo:hi].astype(np.float32)   # fresh state: acc = g
            _, t = O.compress_segment(cfg, acc, part=p, rank=r)
            dec.append(t)
        ref[lo:hi] = O.aggregate(dec, "mean", n)
    assert np.array_equal(res.outs[0], ref)


@pytest.mark.parametrize("kind", ["dgc", "topk"])
@pytest.mark.parametrize("routine", ["alltoall_allgather", "gather_broadcast"])
def test_sparse_process2_recompression(kind, routine):
    """Sparse process 2: partition j of the output is the
    exact top-k_j of q = (rank-order mean of the decoded chunks) + r2 (brute-force
    stable sort), and the second residual obeys the exact sparse EF identity
    transmitted + r2_new == q."""
    n, N = 4, 2500
    cfg = O.Cfg(kind, 0.03, process=2)
    grads = _grads(n, N, dist="D3")   # bf16-rounded: heavy ties
    st = O.new_states(n, N, routine, cfg)
    res = O.sync(routine, cfg, grads, st)
    P = O.nparts_of(routine, n)
    parts = O.partitions(N, P)
    owners = range(n) if routine == "alltoall_allgather" else [0]
    for j, (lo, hi) in zip(owners, parts):
        dec = []
        for r in range(n):
            _, t = O.compress_segment(cfg, grads[r][lo:hi].astype(np.float32), part=j, rank=r)
            dec.append(t)
        q = O.aggregate(dec, "mean", n)               # r2 was 0 before the step
        k = O.k_of(hi - lo, cfg.ratio)
        keys = O.key(q).astype(np.int64)
        order = sorted(range(hi - lo), key=lambda i: (-keys[i], i))[:k]
        sel = np.zeros(hi - lo, bool)
        sel[order] = True
        out = res.outs[0][lo:hi]
        assert np.array_equal(out[sel].view(np.uint32), q[sel].view(np.uint32))
        assert np.all(out[~sel] == 0)
        r2 = st[j].r2
        assert np.array_equal((out + r2).view(np.uint32), q.view(np.uint32))


# ---- the second residual r2 of process 2 (reading R11; P:78-87 Alltoall/
# Allgather, P:105-115 Gather/Broadcast) --------------------------------------
P2_CASES = [(k, r) for k in ("efsignsgd", "onebit", "dgc", "randomk")
            for r in ("alltoall_allgather", "gather_broadcast")]


def _placed_r2(states, routine, N, n):
    """The owners' second residuals placed at their tensor positions (A2A:
    owner j holds partition j; G/B: the root holds the whole tensor)."""
    out = np.zeros(N, np.float64)
    if routine == "alltoall_allgather":
        for j, (lo, hi) in enumerate(O.partitions(N, n)):
            out[lo:hi] = states[j].r2
    else:
        out[:] = states[0].r2
    return out


@pytest.mark.parametrize("kind,routine", P2_CASES)
def test_process2_two_level_ef_telescopes(kind, routine):
    """Two-level error feedback conserves the gradient over T steps.  Per step,
    rank r transmits t1_r = acc_r - r_r,new (first EF); the owner aggregates
    A = mean_r t1_r, adds r2 and transmits t2 = q - r2_new (second EF); every
    rank outputs t2.  Summing over steps telescopes:
        sum_t out_t + r2_T + mean_r r_{r,T} == mean_r sum_t g_{r,t}
    (exact in real arithmetic; here within the fp32 rounding of the adds).
    Dropping r2 from q (q = A) leaves sum_t r2_t instead of r2_T: caught."""
    n, N, T = 4, 1536, 6
    # Randomk: unshared draws, else the second draw repeats the first's support
    # and r2 stays 0 (nothing to pin)
    cfg = O.Cfg(kind, 0.05, process=2, shared_indices=kind != "randomk")
    st = O.new_states(n, N, routine, cfg)
    s_out = np.zeros(N)
    s_g = np.zeros(N)
    mag = 0.0
    for t in range(T):
        grads = [gradient(N, rank=r, step=t, tensor=3) for r in range(n)]
        res = O.sync(routine, cfg, grads, st, tensor_id=3)
        s_out += res.outs[0].astype(np.float64)
        s_g += sum(g.astype(np.float64) for g in grads) / n
        mag = max(mag, max(float(np.abs(g).max()) for g in grads), float(np.abs(res.outs[0]).max()))
    lhs = s_out + _placed_r2(st, routine, N, n) + sum(s.r.astype(np.float64) for s in st) / n
    # each step adds a few fp32 roundings of values <= a few x mag per element
    tol = 8 * T * float(np.spacing(np.float32(4 * mag)))
    assert np.max(np.abs(lhs - s_g)) <= tol
    # r2 must actually be carrying something for the pin to bite
    assert np.abs(_placed_r2(st, routine, N, n)).max() > 100 * tol


def _dyadic(rng, n, lo=-8, hi=8, den=8):
    return (rng.integers(lo, hi + 1, n) / den).astype(np.float32)


@pytest.mark.parametrize("kind", ["efsignsgd", "onebit"])
@pytest.mark.parametrize("routine", ["alltoall_allgather", "gather_broadcast"])
def test_quantized_a7_closed_form_with_nonzero_r2(kind, routine):
    """a7 on an input where every step is exact (P:78-87 / P:105-115 with EF):
    ranks send all-equal magnitudes c_r with random signs, so the first
    compression is lossless (scale = c_r, or class means c_r / -c_r) and the
    owner's aggregate is A = (g_0 + g_1) / 2 exactly.  With a non-zero second
    residual d (dyadic), q = A + d is exact, and the recompression must be the
    closed form scale2 = sum|q| / len (class means for Onebit), bits q >= 0,
    r2_new = q - decode -- computed here in exact rational arithmetic."""
    from fractions import Fraction as F
    n, N = 2, 64
    cfg = O.Cfg(kind, process=2)
    rng = np.random.default_rng(7)
    signs = [np.where(rng.random(N) < 0.5, -1.0, 1.0).astype(np.float32) for _ in range(n)]
    grads = [signs[0] * np.float32(1.0), signs[1] * np.float32(0.5)]
    st = O.new_states(n, N, routine, cfg)
    parts = O.partitions(N, n) if routine == "alltoall_allgather" else [(0, N)]
    owners = list(range(n)) if routine == "alltoall_allgather" else [0]
    d_full = _dyadic(rng, N)
    for j, (lo, hi) in zip(owners, parts):
        st[j].r2 = d_full[lo:hi].copy()
    res = O.sync(routine, cfg, grads, st)
    for j, (lo, hi) in zip(owners, parts):
        A = [(F(float(grads[0][i])) + F(float(grads[1][i]))) / 2 for i in range(lo, hi)]
        q = [a + F(float(d_full[i])) for a, i in zip(A, range(lo, hi))]
        if kind == "efsignsgd":
            s = sum(abs(x) for x in q) / len(q)
            dec = [s if x >= 0 else -s for x in q]
        else:
            pos = [x for x in q if x >= 0]
            neg = [x for x in q if x < 0]
            mp = sum(pos) / len(pos) if pos else F(0)
            mn = sum(neg) / len(neg) if neg else F(0)
            dec = [mp if x >= 0 else mn for x in q]
        # decoded values are exactly representable here (dyadic / 32 or / class size
        # rounded once to fp32): compare in fp32
        want = np.array([float(x) for x in dec], np.float32)
        assert np.array_equal(res.outs[0][lo:hi], want), (j, kind, routine)
        want_r2 = np.array([float(x) for x in q], np.float32) - want
        assert np.array_equal(st[j].r2, want_r2.astype(np.float32))


# ---- hierarchical communication (reading R23) ------
HIER = [("dgc", "allgather"), ("dgc", "alltoall_allgather"), ("randomk", "gather_broadcast"),
        ("efsignsgd", "alltoall_allgather"), ("onebit", "allgather"), ("topk", "gather_broadcast")]


@pytest.mark.parametrize("kind,routine", HIER)
def test_hier_one_gpu_per_machine_is_flat(kind, routine):
    """g = 1: the intra-machine phases are identities and the inter-machine
    phase is the flat routine over all n ranks (flat = one phase)."""
    n, N = 4, 3001
    cfg = O.Cfg(kind, 0.02)
    grads = _grads(n, N)
    h = O.sync_hierarchical(routine, cfg, grads, O.new_states_hier(n, N, routine, cfg, 1), 1, tensor_id=5)
    f = O.sync(routine, cfg, grads, O.new_states(n, N, routine, cfg), tensor_id=O.hier_shard_tensor_id(5, 0))
    for r in range(n):
        assert np.array_equal(h.outs[r], f.outs[r])


@pytest.mark.parametrize("n,g", [(4, 2), (8, 4), (8, 2), (6, 3), (4, 4)])
@pytest.mark.parametrize("kind", ["dgc", "randomk"])
def test_hier_rho1_is_the_global_mean(n, g, kind):
    """rho = 1: nothing is dropped, so after the three phases every rank holds
    the mean of all n gradients (mean of the machines' means), within the
    fp32 rounding of two averaging stages -- pins which shard goes where."""
    N = 2999
    cfg = O.Cfg(kind, 1.0)
    grads = _grads(n, N, dist="D2")
    res = O.sync_hierarchical("allgather", cfg, grads, O.new_states_hier(n, N, "allgather", cfg, g), g)
    x = np.stack([gg.astype(np.float64) for gg in grads])
    exact, scale = x.mean(0), np.abs(x).mean(0)
    for r in range(n):
        assert np.all(np.abs(res.outs[r].astype(np.float64) - exact) <= 4e-7 * scale + 1e-38)


@pytest.mark.parametrize("kind,routine", HIER)
@pytest.mark.parametrize("n,g", [(4, 2), (8, 4)])
def test_hier_bytes_closed_form(kind, routine, n, g):
    """Per rank: the intra Reduce-scatter and Allgather each receive the other
    g-1 shards (4 (g-1) N / g bytes up to partition rounding), and the
    inter-machine phase moves the cost-table volume of the routine for the
    shard's payload over m = n / g ranks."""
    N = 8192
    cfg = O.Cfg(kind, 0.02)
    res = O.sync_hierarchical(routine, cfg, _grads(n, N), O.new_states_hier(n, N, routine, cfg, g), g)
    m = n // g
    L = O.partitions(N, g)[0][1]
    P = O.nparts_of(routine, m)
    M = O.chunk_bytes(cfg, L, P) * P
    row = O.table_row(cfg, routine)
    c = res.counters[0]   # rank (0, 0): root of its inter group
    ph = {name: (s, rcv) for name, s, rcv in c.phases}
    assert ph["intra_reducescatter"][1] == 4 * L * (g - 1)
    assert ph["intra_allgather"][1] == 4 * (N - L)
    inter_recv = ph["inter_" + routine][1]
    if routine != "gather_broadcast":
        assert inter_recv == pytest.approx(O.table_comm_bytes(row, M, m), abs=m)


@pytest.mark.parametrize("kind", ["dgc", "randomk"])
def test_hier_ef_telescopes(kind):
    """Error feedback lives per (machine, shard): over T steps the output plus
    the machines' mean residual of each shard equals the sum of the global
    mean gradients (within fp32 rounding)."""
    n, g, N, T = 8, 4, 4000, 5
    cfg = O.Cfg(kind, 0.05, shared_indices=False)
    st = O.new_states_hier(n, N, "allgather", cfg, g)
    s_out, s_g = np.zeros(N), np.zeros(N)
    mag = 0.0
    for t in range(T):
        grads = [gradient(N, rank=r, step=t) for r in range(n)]
        res = O.sync_hierarchical("allgather", cfg, grads, st, g)
        s_out += res.outs[0].astype(np.float64)
        s_g += sum(gg.astype(np.float64) for gg in grads) / n
        mag = max(mag, max(float(np.abs(gg).max()) for gg in grads))
    resid = np.zeros(N)
    for i, (lo, hi) in enumerate(O.partitions(N, g)):
        resid[lo:hi] = sum(st[a * g + i].r.astype(np.float64) for a in range(n // g)) / (n // g)
    tol = 16 * T * float(np.spacing(np.float32(4 * mag)))
    assert np.max(np.abs(s_out + resid - s_g)) <= tol
    assert np.abs(resid).max() > 100 * tol
