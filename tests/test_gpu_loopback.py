"""The fused collectives of a real n-rank job on ONE GPU (loopback group,
esp_world_create_loopback): n worlds act as ranks 0..n-1 with the real ranks'
push-job tables, slot layouts, arrival counters and both call parities, over
plain device pointers instead of CUDA IPC, every kernel on one stream in
dependency order (no kernel waits for a later one).  Every rank's output and
EF state is compared with the oracle's n-rank simulation (SURVEY.md 8a a6,
8f NEXT-1) -- the 8-rank layout is checked on a single B200."""
import numpy as np
import pytest

from oracle import esp_oracle as O
from synth.values import gradient

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import __graft_entry__
    __graft_entry__.build()


def E():
    from paper_2205_14465_b200 import esp
    return esp


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def check(kind, got, ref, where):
    if kind in O.QUANTIZED:
        np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-30, err_msg=where)
    else:
        bad = np.nonzero(bits(got) != bits(ref))[0]
        assert bad.size == 0, f"{where}: {bad.size} mismatches at {bad[:5]}"


# every fused (byte-moving) routine x process x compressor
CASES = [(k, "allgather", 0, sh) for k, sh in (("dgc", True), ("topk", True), ("randomk", True), ("randomk", False),
                                               ("efsignsgd", True), ("onebit", True))]
CASES += [(k, r, p, sh) for r in ("alltoall_allgather", "gather_broadcast") for p in (1, 2)
          for k, sh in (("dgc", True), ("topk", True), ("randomk", True), ("randomk", False),
                        ("efsignsgd", True), ("onebit", True))]


def run_group(n, specs, steps=3, ratio=0.02, seed=5):
    """specs: [(kind, routine, process, shared, N)], one ctx per spec per rank,
    all synchronised together with esp_sync_many_loopback for `steps` steps."""
    e = E()
    ws = e.World.loopback(n, 0)
    try:
        ctxs = [[e.Ctx(ws[r], k, ro, N, tensor_id=50 + i, ratio=ratio, process=p, shared_indices=sh, seed=seed)
                 for i, (k, ro, p, sh, N) in enumerate(specs)] for r in range(n)]
        cfgs = [O.Cfg(k, ratio, seed=seed, shared_indices=sh, process=p) for (k, ro, p, sh, N) in specs]
        sts = [O.new_states(n, N, ro, cfgs[i]) for i, (k, ro, p, sh, N) in enumerate(specs)]
        for s in range(steps):
            for i, (k, ro, p, sh, N) in enumerate(specs):
                if k in O.QUANTIZED and s > 0:   # lock-step: oracle state -> GPU (never the reverse)
                    for r in range(n):
                        r2len = ctxs[r][i].get_state()[2].shape[1]
                        r2 = np.zeros((1, r2len), np.float32)
                        if sts[i][r].r2 is not None:
                            r2[0, :sts[i][r].r2.size] = sts[i][r].r2
                        ctxs[r][i].set_state(sts[i][r].step, sts[i][r].r[None], r2)
            grads = [[gradient(N, step=s, rank=r, tensor=50 + i) for r in range(n)]
                     for i, (_, _, _, _, N) in enumerate(specs)]
            refs = [O.sync(ro, cfgs[i], grads[i], sts[i], tensor_id=50 + i) for i, (k, ro, p, sh, N) in enumerate(specs)]
            dev = [[torch.from_numpy(grads[i][r].copy()).cuda() for i in range(len(specs))] for r in range(n)]
            e.esp_sync_many_loopback(ws, ctxs, dev)
            torch.cuda.synchronize()
            for w in ws:
                w.check()   # every wait kernel found its arrivals complete
            for i, (k, ro, p, sh, N) in enumerate(specs):
                for r in range(n):
                    where = f"n={n} {k}/{ro}/p{p}/shared={sh} N={N} step={s} rank={r}"
                    check(k, dev[r][i].cpu().numpy(), refs[i].outs[r], where + " out")
                    _, rg, r2g = ctxs[r][i].get_state()
                    if k in O.QUANTIZED:
                        np.testing.assert_allclose(rg[0], sts[i][r].r, rtol=1e-6, atol=1e-30, err_msg=where + " r")
                    else:
                        assert np.array_equal(bits(rg[0]), bits(sts[i][r].r)), where + " residual"
                        if sts[i][r].r2 is not None:
                            assert np.array_equal(bits(r2g[0, :sts[i][r].r2.size]), bits(sts[i][r].r2)), where + " r2"
    finally:
        for w in ws:
            w.destroy()


@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("kind,routine,process,shared", CASES)
def test_loopback_pair(n, kind, routine, process, shared):
    run_group(n, [(kind, routine, process, shared, 30_011)])


@pytest.mark.parametrize("n", [4, 8])
def test_loopback_mixed_buckets(n):
    """A mixed strategy (several buckets, tensors smaller than n x 32 with empty
    partitions, both processes) over 4 steps: both call parities twice."""
    specs = [("dgc", "allgather", 0, True, 70_001), ("efsignsgd", "alltoall_allgather", 0, True, 9000),
             ("dgc", "alltoall_allgather", 0, True, 40_000), ("onebit", "gather_broadcast", 0, True, 5000),
             ("dgc", "allgather", 0, True, 33), ("efsignsgd", "alltoall_allgather", 0, True, 40),
             ("dgc", "alltoall_allgather", 2, True, 50), ("randomk", "alltoall_allgather", 2, False, 3000),
             ("topk", "gather_broadcast", 2, True, 77), ("efsignsgd", "alltoall_allgather", 1, True, 6000),
             ("randomk", "gather_broadcast", 1, True, 2048)]
    run_group(n, specs, steps=4, ratio=0.01)


def test_loopback_rejects_nccl_reduced_buckets():
    e = E()
    ws = e.World.loopback(2, 0)
    try:
        ctxs = [[e.Ctx(ws[r], "none", "allreduce", 100, tensor_id=0)] for r in range(2)]
        g = [[torch.zeros(100, device="cuda")] for _ in range(2)]
        with pytest.raises(e.EspError):
            e.esp_sync_many_loopback(ws, ctxs, g)
        with pytest.raises(e.EspError):
            e.esp_sync(ws[0], ctxs[0][0], g[0][0])
    finally:
        for w in ws:
            w.destroy()
