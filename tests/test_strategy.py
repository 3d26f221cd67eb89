"""NEXT-3 strategy selection (no GPU): the C ABI's curve fit, per-option time
and GetBestOption against the oracle's, and both against closed forms of the
cost table and the curve-fit examples."""
import math
import random

import pytest

from oracle import esp_oracle as O

E = pytest.importorskip("paper_2205_14465_b200.esp")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import __graft_entry__
    __graft_entry__.build()


CURVE = [(2 ** 20, 100e-6), (2 ** 30, 10e-3)]


@pytest.mark.parametrize("nbytes,expect", [(2 ** 20, 100e-6), (2 ** 25, 1e-3), (2 ** 10, 100e-6),
                                           (2 ** 31, 10e-3 * 10 ** 0.2)])
def test_curve_fit_examples(nbytes, expect):
    # exact sample point; log-log midpoint = geometric mean; clamp below the
    # first sample; above the last, the last segment's slope (10^0.2 per doubling)
    assert O.curve_eval(CURVE, nbytes) == pytest.approx(expect, rel=1e-12)
    assert E.curve_eval(CURVE, nbytes) == pytest.approx(expect, rel=1e-12)


def test_curve_errors():
    with pytest.raises(E.EspError):
        E.curve_eval([(2.0, 1.0), (1.0, 2.0)], 1.5)
    with pytest.raises(E.EspError):
        E.curve_eval([(1.0, 0.0)], 1.0)


def test_option_time_closed_form():
    # constant 1 ms curves: Allgather n = 4 -> h1 + 4 h2 = 5 ms plus
    # (n-1) M / B of communication
    one = [(1.0, 1e-3)]
    N, n, B = 1_000_000, 4, 1.25e10
    cfg = O.Cfg("dgc", 0.01)
    M = O.chunk_bytes(cfg, N, 1)
    want = 5e-3 + 3 * M / B
    assert O.option_time(cfg, "allgather", N, n, B, one, one) == pytest.approx(want, rel=1e-12)
    o = E.make_option("dgc", 0.01, "allgather", h1=one, h2=one)
    assert E.option_time(o, N, n, B) == pytest.approx(want, rel=1e-12)
    # uncompressed: only 2(n-1)M/(nB) of communication
    assert E.option_time(E.make_option("none", 1.0, "allreduce"), N, n, B) == pytest.approx(
        2 * 3 * 4 * N / 4 / B, rel=1e-12)


@pytest.mark.parametrize("routine,ms", [("allreduce", 12.0), ("reducescatter_allgather", 12.0),
                                        ("reduce_broadcast", 32.0)])
def test_uncompressed_routine_times_spec_examples(routine, ms):
    """Per-step volumes of S:126 at n = 4, M = 1e8 B, B = 1.25e10 B/s:
    Allreduce 2(n-1)M/(nB) = 12 ms; Reduce-scatter (n-1)M/(nB) = 6 ms + Allgather
    of the shards 6 ms; Reduce (n-1)M/B = 24 ms + Broadcast of the M-byte result
    M/B = 8 ms."""
    N, n, B = 25_000_000, 4, 1.25e10
    assert O.option_time(O.Cfg("none", 1.0), routine, N, n, B, None, None) == pytest.approx(ms * 1e-3, rel=1e-12)
    assert E.option_time(E.make_option("none", 1.0, routine), N, n, B) == pytest.approx(ms * 1e-3, rel=1e-12)


def _random_curve(rng):
    xs = sorted({2 ** rng.randint(8, 30) for _ in range(6)})
    t, out = rng.uniform(5e-6, 5e-5), []
    for x in xs:
        t *= rng.uniform(1.0, 3.0)
        out.append((float(x), t))
    return out


OPTS = [("none", "allreduce", 0), ("none", "reduce_broadcast", 0), ("none", "reducescatter_allgather", 0), ("randomk", "allreduce", 0), ("dgc", "allgather", 0),
        ("dgc", "alltoall_allgather", 1), ("dgc", "alltoall_allgather", 2), ("dgc", "gather_broadcast", 1),
        ("dgc", "gather_broadcast", 2), ("efsignsgd", "allgather", 0), ("efsignsgd", "alltoall_allgather", 2),
        ("onebit", "gather_broadcast", 2), ("randomk", "alltoall_allgather", 1)]


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_option_time_and_selection_match_oracle(n):
    rng = random.Random(7 + n)
    for trial in range(30):
        N = rng.choice([1000, 4096, 100_003, 2 ** 20, 3 * 2 ** 20, 25_000_000])
        B = 10 ** rng.uniform(8, 12)
        opts_e, opts_o = [], []
        for kind, routine, proc in OPTS:
            h1, h2 = _random_curve(rng), _random_curve(rng)
            ratio = rng.choice([0.001, 0.01, 0.1]) if kind in O.SPARSE else 1.0
            opts_e.append(E.make_option(kind, ratio, routine, h1=h1, h2=h2, process=proc))
            opts_o.append((O.Cfg(kind, ratio, process=proc), routine, h1, h2))
            te = E.option_time(opts_e[-1], N, n, B)
            to = O.option_time(opts_o[-1][0], routine, N, n, B, h1, h2)
            assert te == pytest.approx(to, rel=1e-9), (kind, routine, proc, N, n)
        be, tbe = E.select_option(opts_e, N, n, B)
        bo, tbo = O.select_option(opts_o, N, n, B)
        assert be == bo and tbe == pytest.approx(tbo, rel=1e-9)


def test_selection_limits():
    """Unbounded bandwidth: no compression wins (it has no compression time);
    a vanishing bandwidth: the smallest payload (1 bit per element) wins."""
    cur = [(1024.0, 1e-5), (2.0 ** 30, 1e-3)]
    opts = [E.make_option("none", 1.0, "allreduce"), E.make_option("dgc", 0.01, "allgather", h1=cur, h2=cur),
            E.make_option("efsignsgd", 1.0, "alltoall_allgather", h1=cur, h2=cur)]
    assert E.select_option(opts, 10_000_000, 8, 1e18)[0] == 0
    assert E.select_option(opts, 10_000_000, 8, 1e3)[0] == 2
