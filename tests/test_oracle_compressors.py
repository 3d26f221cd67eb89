"""Pins of the oracle's compressors against brute force, closed forms and
invariants (no GPU).  Each pin is independent of the oracle's own code path:
brute force enumerates subsets / uses heapq / math.fsum / per-bit loops."""
import heapq
import itertools
import math

import numpy as np
import pytest

from oracle import esp_oracle as O
from synth.values import gradient, D4_MODES


def _tuple_order(x):
    k = [struct_key(v) for v in x]
    return k


def struct_key(v):
    # |v| ordering by bit pattern of a float32, computed via Python struct (independent of O.key)
    import struct
    return struct.unpack("<I", struct.pack("<f", float(np.float32(v))))[0] & 0x7FFFFFFF


# ---------------------------------------------------------------- top-k / DGC
@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 8])
def test_topk_brute_force_subsets(n):
    """Brute force: the top-k set S is the unique k-subset whose every member
    precedes every non-member in (key desc, idx asc) order (R2)."""
    rng = np.random.default_rng(n)
    vals = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, 2.0, 0.5, -2.0], np.float32), n)
    keys = [struct_key(v) for v in vals]
    for k in range(1, n + 1):
        got = set(O.topk_select(vals, k).tolist())
        found = []
        for S in itertools.combinations(range(n), k):
            S = set(S)
            ok = all((keys[i] > keys[j]) or (keys[i] == keys[j] and i < j)
                     for i in S for j in range(n) if j not in S)
            if ok:
                found.append(S)
        assert len(found) == 1
        assert got == found[0]


@pytest.mark.parametrize("dist", ["D1", "D2", "D3"])
@pytest.mark.parametrize("n,ratio", [(1000, 0.01), (4097, 0.001), (33, 0.5), (20000, 0.01)])
def test_topk_vs_heap(dist, n, ratio):
    g = gradient(n, dist=dist)
    k = O.k_of(n, ratio)
    keys = [struct_key(v) for v in g]
    ref = sorted(heapq.nsmallest(k, range(n), key=lambda i: (-keys[i], i)))
    assert O.topk_select(g, k).tolist() == ref


@pytest.mark.parametrize("mode", D4_MODES)
def test_topk_adversarial(mode):
    g = gradient(3001, dist="D4", mode=mode)
    k = O.k_of(g.size, 0.01)
    keys = [struct_key(v) for v in g]
    ref = sorted(heapq.nsmallest(k, range(g.size), key=lambda i: (-keys[i], i)))
    assert O.topk_select(g, k).tolist() == ref


def test_topk_all_equal_takes_first_indices():
    g = np.full(100, -3.0, np.float32)
    g[::2] = 3.0
    assert O.topk_select(g, 7).tolist() == list(range(7))


def test_k_rounding():
    # R1: k = min(N, max(1, ceil(rho N)))
    assert O.k_of(2 ** 20, 0.01) == 10486
    assert O.k_of(10 ** 6, 0.01) == 10000
    assert O.k_of(5, 0.001) == 1
    assert O.k_of(7, 1.0) == 7
    assert O.k_of(0, 0.5) == 0


def test_sparse_ef_invariant_exact():
    """transmitted + r_new == acc, value for value (SURVEY 8c 'Sparse EF')."""
    for dist in ("D1", "D3"):
        acc = gradient(5000, dist=dist)
        for kind in ("dgc", "randomk"):
            ch, t = O.compress_segment(O.Cfg(kind, 0.01), acc)
            r = O.residual_update(acc, t)
            assert np.array_equal((t + r).astype(np.float32), acc)
            assert np.all(r[ch.idx.astype(int)] == 0)
            mask = np.ones(acc.size, bool)
            mask[ch.idx.astype(int)] = False
            assert np.array_equal(r[mask].view(np.uint32), acc[mask].view(np.uint32))


# ---------------------------------------------------------------- randomk
def test_randomk_strata_invariants():
    for N, k in [(100, 10), (1000, 7), (33, 33), (2 ** 20 + 3, 10487), (5, 1)]:
        idx = O.randomk_indices(N, k, 1, 2, 3, 0, None).astype(np.int64)
        assert idx.size == k
        assert np.all(np.diff(idx) > 0)
        assert idx.min() >= 0 and idx.max() < N
        # one per stratum [floor(jN/k), floor((j+1)N/k)) — checked with Python ints
        for j in range(0, k, max(1, k // 50)):
            assert (j * N) // k <= idx[j] < ((j + 1) * N) // k


def test_randomk_deterministic_and_shared():
    a = O.randomk_indices(1000, 10, 5, 1, 2, 0, None)
    b = O.randomk_indices(1000, 10, 5, 1, 2, 0, None)
    assert np.array_equal(a, b)
    c = O.randomk_indices(1000, 10, 5, 1, 3, 0, None)
    assert not np.array_equal(a, c)            # step changes the draw
    r0 = O.randomk_indices(1000, 10, 5, 1, 2, 0, 0)
    r1 = O.randomk_indices(1000, 10, 5, 1, 2, 0, 1)
    assert not np.array_equal(r0, r1)          # per-rank draw when not shared


def test_randomk_chi_square_uniform():
    """Each index is selected with frequency k/N (chi-square over 4000 draws)."""
    N, k, T = 64, 8, 4000
    counts = np.zeros(N)
    for s in range(T):
        counts[O.randomk_indices(N, k, s, 0, 0, 0, None).astype(int)] += 1
    expected = T * k / N
    chi2 = ((counts - expected) ** 2 / expected).sum()
    # 63 dof; p=0.001 critical value ~ 103
    assert chi2 < 103


def test_splitmix64_known_value():
    # splitmix64 reference sequence from seed 0: first output 0xE220A8397B1DCDAF
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF
    assert int(O.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF


# ---------------------------------------------------------------- sign / onebit
def test_pack_bits_per_bit_loop():
    rng = np.random.default_rng(0)
    for n in (1, 31, 32, 33, 100):
        bits = rng.integers(0, 2, n).astype(bool)
        words = O.pack_bits(bits)
        assert words.size == -(-n // 32)
        for i in range(n):
            assert ((int(words[i // 32]) >> (i % 32)) & 1) == int(bits[i])
        for i in range(n, words.size * 32):
            assert ((int(words[i // 32]) >> (i % 32)) & 1) == 0
        assert np.array_equal(O.unpack_bits(words, n), bits)


def test_exact_sum_vs_fsum():
    for dist in ("D1", "D2", "D3"):
        x = gradient(10001, dist=dist)
        assert O.f64(O.exact_sum(x)) == math.fsum(float(v) for v in x)
    x = gradient(1000, dist="D4", mode="denormal")
    assert O.f64(O.exact_sum(x)) == math.fsum(float(v) for v in x)


def test_sign_scale_closed_form_and_ef():
    # all |p| = c -> scale = c, transmitted == p, r_new == 0
    c = np.float32(0.37)
    p = np.where(np.arange(777) % 3 == 0, c, -c).astype(np.float32)
    ch, t = O.compress_segment(O.Cfg("efsignsgd"), p)
    assert ch.scale == c
    assert np.array_equal(t, p)
    assert np.all(O.residual_update(p, t) == 0)


@pytest.mark.parametrize("kind", ["efsignsgd", "onebit"])
@pytest.mark.parametrize("dist", ["D1", "D2", "D3"])
def test_sign_ef_half_ulp(kind, dist):
    acc = gradient(4099, dist=dist)
    ch, t = O.compress_segment(O.Cfg(kind), acc)
    r = O.residual_update(acc, t)
    err = np.abs(t.astype(np.float64) + r.astype(np.float64) - acc.astype(np.float64))
    half_ulp = np.spacing(np.abs(r)).astype(np.float64) / 2
    assert np.all(err <= half_ulp)
    if kind == "efsignsgd":
        ref = np.float32(math.fsum(abs(float(v)) for v in acc) / acc.size)
        assert ch.scale == ref
        assert np.array_equal(O.unpack_bits(ch.words, acc.size), acc >= 0)
    else:
        pos = acc >= 0
        assert ch.mpos == np.float32(math.fsum(float(v) for v in acc[pos]) / pos.sum())
        assert ch.mneg == np.float32(math.fsum(float(v) for v in acc[~pos]) / (~pos).sum())


def test_sign_zero_conventions():
    # R6: bit = (p >= 0): +0 and -0 -> 1
    p = np.array([0.0, -0.0, -1.0, 1.0], np.float32)
    ch, _ = O.compress_segment(O.Cfg("efsignsgd"), p)
    assert O.unpack_bits(ch.words, 4).tolist() == [True, True, False, True]
    ch, _ = O.compress_segment(O.Cfg("onebit"), np.array([1.0, 3.0], np.float32))
    assert ch.mneg == 0 and ch.mpos == 2.0          # empty class -> 0


# ---------------------------------------------------------------- sizes
def test_compressed_sizes_spec_examples():
    # sparsification rho=0.01, M=4e8 B (1e8 fp32) -> 8e6 B
    assert O.chunk_bytes(O.Cfg("dgc", 0.01), 10 ** 8, 1) == 8_000_000
    # 1-bit, M=4e8 B -> 12,500,000 B of words; this build's header is 16 B (R18b)
    assert O.chunk_bytes(O.Cfg("efsignsgd"), 10 ** 8, 1) == 12_500_000 + 16
    # rho = 1 -> 2M
    assert O.chunk_bytes(O.Cfg("dgc", 1.0), 1000, 1) == 2 * 4000
    # 1-bit saves 96.9%: 1/32 of the fp32 bytes, up to the header
    b = O.chunk_bytes(O.Cfg("efsignsgd"), 2 ** 24, 1)
    assert abs(1 - b / (4 * 2 ** 24) - 0.969) < 0.001


def test_partitions():
    assert O.partitions(100, 1) == [(0, 100)]
    p = O.partitions(1000, 8)        # L = ceil(125/32)*32 = 128
    assert p[0] == (0, 128) and p[7] == (896, 1000)
    p = O.partitions(33, 4)          # L = 32: [0,32),[32,33),[33,33),[33,33)
    assert p == [(0, 32), (32, 33), (33, 33), (33, 33)]
    for N in (1, 31, 1000, 12345):
        for n in (2, 4, 8):
            parts = O.partitions(N, n)
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


# ---- DGC momentum correction (R20) -----------------------------------------
def test_momentum_zero_is_plain_dgc():
    N, n = 20_000, 2
    a, b = O.Cfg("dgc", 0.01), O.Cfg("dgc", 0.01, momentum=0.0)
    sa, sb = O.new_states(n, N, "allgather", a), O.new_states(n, N, "allgather", b)
    for s in range(3):
        grads = [gradient(N, step=s, rank=r) for r in range(n)]
        ra = O.sync("allgather", a, grads, sa)
        rb = O.sync("allgather", b, grads, sb)
        assert np.array_equal(ra.outs[0], rb.outs[0])


def test_momentum_geometric_series_closed_form():
    """A coordinate that is never selected, under a constant gradient c, obeys
    u_t = c (1 - m^(t+1)) / (1 - m) and v_t = sum_{s<=t} u_s.  With m = 1/2 and
    c = 2^-20 every term is exact in fp32, so the oracle must match exactly;
    a dominant spike keeps the coordinate unselected (k = 1)."""
    N, m, c, T = 64, 0.5, 2.0 ** -20, 12
    cfg = O.Cfg("dgc", 1 / 64, momentum=m)   # k = 1
    st = O.new_states(1, N, "allgather", cfg)
    v = 0.0
    for t in range(T):
        g = np.full(N, c, np.float32)
        g[0] = 1.0                      # selected every step (largest by far)
        O.sync("allgather", cfg, [g], st)
        u = c * (1 - m ** (t + 1)) / (1 - m)
        v += u
        assert st[0].u[5] == np.float32(u)
        assert st[0].r[5] == np.float32(v)
        assert st[0].u[0] == 0 and st[0].r[0] == 0   # momentum factor masking


def test_momentum_rho1_is_uncompressed_mean():
    """rho = 1: every coordinate is sent and both u and v are reset each step,
    so the output is the plain mean of the gradients whatever m is."""
    n, N = 3, 1000
    cfg = O.Cfg("dgc", 1.0, momentum=0.9)
    st = O.new_states(n, N, "allgather", cfg)
    for s in range(3):
        grads = [gradient(N, step=s, rank=r) for r in range(n)]
        res = O.sync("allgather", cfg, grads, st)
        assert np.array_equal(res.outs[0], O.aggregate(grads, "mean", n))
        assert all(np.all(x.u == 0) and np.all(x.r == 0) for x in st)


def test_momentum_ef_identity_and_masking():
    """transmitted + v_new == fl(u_new_unmasked + v_old) bit for bit, and
    u_new is zero exactly on the selected support."""
    N = 30_000
    cfg = O.Cfg("dgc", 0.01, momentum=0.9)
    st = O.new_states(1, N, "allgather", cfg)
    for s in range(4):
        g = gradient(N, step=s, dist="D3")
        u_pred = (np.float32(0.9) * st[0].u).astype(np.float32)
        u_pred = (u_pred + g).astype(np.float32)
        acc = (u_pred + st[0].r).astype(np.float32)
        res = O.sync("allgather", cfg, [g], st)
        out, v = res.outs[0], st[0].r
        assert np.array_equal((out + v).view(np.uint32), acc.view(np.uint32))
        sel = np.zeros(N, bool)
        sel[O.topk_select(acc, O.k_of(N, 0.01)).astype(np.int64)] = True
        assert np.all(st[0].u[sel] == 0)
        assert np.array_equal(st[0].u[~sel].view(np.uint32), u_pred[~sel].view(np.uint32))


# ---------------------------------------------------------------- approximate-count DGC (R22)
def _py_splitmix(z):
    z = (z + 0x9E3779B97F4A7C15) % 2 ** 64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % 2 ** 64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % 2 ** 64
    return z ^ (z >> 31)


@pytest.mark.parametrize("n,rate", [(4097, 0.0), (5000, 0.0), (100_003, 0.0), (1 << 20, 0.0), (100_003, 0.01),
                                    (1 << 20, 0.001), (9000, 0.5)])
def test_dgc_sample_positions_strata(n, rate):
    """Each of the S strata [floor(Gn/S), floor((G+1)n/S)) contributes 8
    consecutive in-range positions at the offset its hash gives -- recomputed
    with Python integers (not numpy uint64).  S = 512, or ceil(rate n / 8)
    capped at 512."""
    h = O.dgc_segment_hash(7, 1)
    S = 512 if rate == 0 else min(512, max(1, -(-int(rate * n * 1000) // 8000)))
    assert O.dgc_strata(n, rate) == S
    pos = O.dgc_sample_positions(n, h, S)
    assert pos.size == 8 * S
    for G in range(S):
        a, b = G * n // S, (G + 1) * n // S
        off = ((_py_splitmix(h ^ G) & 0xFFFFFFFF) * (b - a - 7)) >> 32
        want = [a + off + c for c in range(8)]
        assert list(pos[8 * G:8 * G + 8]) == want
        assert a <= want[0] and want[-1] < b
    assert np.all(np.diff(pos) > 0)


@pytest.mark.parametrize("approx", [False, True])
@pytest.mark.parametrize("ratio", [0.001, 0.01])
def test_dgc_threshold_is_prefix_of_sampled_rank(approx, ratio):
    """The threshold is the need-th largest sampled key with its low 10 bits
    cleared; recomputed with Python's sorted() over struct-derived keys."""
    n = 300_001
    acc = gradient(n, dist="D2")
    k = O.k_of(n, ratio)
    h = O.dgc_segment_hash(3, 0)
    thr = O.dgc_threshold(acc, k, ratio, h, approx)
    pos = O.dgc_sample_positions(n, h)
    keys = sorted((struct_key(acc[p]) for p in pos), reverse=True)
    rs = ratio * 4096
    need = int(rs + 0.5) if approx else math.ceil(rs + 4 * math.sqrt(rs))
    assert thr == keys[need - 1] // 1024 * 1024


@pytest.mark.parametrize("dist", ["D1", "D2", "D3"])
@pytest.mark.parametrize("ratio", [0.001, 0.01, 0.1])
def test_dgc_approx_is_top_m(dist, ratio):
    """Approximate-count DGC keeps m = min(k, #{key >= thr}) elements, and they
    are the top-m in (key desc, idx asc) order: the brute-force stable sort's
    first m; the sparse EF identity holds exactly."""
    n = 100_003
    acc = gradient(n, dist=dist, tensor=5)
    cfg = O.Cfg("dgc", ratio, approx=True)
    k = O.k_of(n, ratio)
    thr = O.dgc_threshold(acc, k, ratio, O.dgc_segment_hash(5, 0), True)
    ch, t = O.compress_segment(cfg, acc, tensor_id=5)
    keys = np.array([struct_key(v) for v in acc], np.int64)   # struct-derived, not O.key
    m = min(k, int((keys >= thr).sum()))
    order = sorted(range(n), key=lambda i: (-keys[i], i))[:m]
    assert ch.idx.size == m
    assert np.array_equal(ch.idx, np.sort(np.array(order, np.uint32)))
    r = O.residual_update(acc, t)
    assert np.array_equal((t + r).view(np.uint32), acc.view(np.uint32))


def test_dgc_approx_count_unbiased():
    """With the expected rank j* = round(rho s), the number kept averages about
    k over many independent segments (the sampled threshold is unbiased up to
    the bin rounding), and is capped at k."""
    n, ratio = 60_000, 0.01
    k = O.k_of(n, ratio)
    counts = []
    for t in range(150):
        acc = gradient(n, tensor=t)
        ch, _ = O.compress_segment(O.Cfg("dgc", ratio, approx=True), acc, tensor_id=t)
        counts.append(ch.idx.size)
    counts = np.array(counts)
    assert counts.max() <= k
    # capped at k, the mean sits a little below k; uncapped it would be ~k
    assert 0.80 * k < counts.mean() <= k


def test_dgc_approx_small_segments_are_exact():
    """Segments of <= 4096 elements are their own sample with need = k: the
    approximate mode returns the exact top-k."""
    for n, ratio in ((33, 0.1), (1000, 0.01), (4096, 0.05)):
        acc = gradient(n, dist="D3")
        a, _ = O.compress_segment(O.Cfg("dgc", ratio, approx=True), acc)
        assert np.array_equal(a.idx, O.topk_select(acc, O.k_of(n, ratio)))
