"""Hierarchical communication (reading R23) on
one GPU: a loopback group of n ranks forming n / g "machines" of g GPUs
(esp_world_create_loopback_hier) runs the three phases -- intra-machine
Reduce-scatter pushed over device pointers, the inter-machine compressed
routine of each shard (the flat fused engine on the shard's group), the
intra-machine Allgather -- with every kernel in dependency order on one
stream.  Every rank's output and its shard's EF state against the oracle's
sync_hierarchical, bit-exact where the arithmetic is fixed (sign scales 1e-6
relative, lock-stepped)."""
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


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def run(n, g, specs, steps=3, ratio=0.02):
    from paper_2205_14465_b200 import esp as E
    ws = E.World.loopback_hier(n, g, 0)
    try:
        ctxs = [[E.Ctx(ws[r], k, ro, N, tensor_id=60 + i, ratio=ratio, process=p) for i, (k, ro, p, N) in enumerate(specs)]
                for r in range(n)]
        cfgs = [O.Cfg(k, ratio, process=p) for (k, ro, p, N) in specs]
        sts = [O.new_states_hier(n, N, ro, cfgs[i], g) for i, (k, ro, p, N) in enumerate(specs)]
        for s in range(steps):
            for i, (k, ro, p, N) in enumerate(specs):
                if k in O.QUANTIZED and s > 0:   # lock-step: oracle state -> GPU
                    for r in range(n):
                        st = sts[i][r]
                        if st.r.size == 0:
                            continue   # this rank's shard of the tensor is empty
                        r2len = ctxs[r][i].get_state()[2].shape[1]
                        r2 = np.zeros((1, r2len), np.float32)
                        if st.r2 is not None:
                            r2[0, :st.r2.size] = st.r2
                        ctxs[r][i].set_state(st.step, st.r[None], r2)
            grads = [[gradient(N, step=s, rank=r, tensor=60 + i) for r in range(n)]
                     for i, (_, _, _, N) in enumerate(specs)]
            refs = [O.sync_hierarchical(ro, cfgs[i], grads[i], sts[i], g, tensor_id=60 + i)
                    for i, (k, ro, p, N) in enumerate(specs)]
            dev = [[torch.from_numpy(grads[i][r].copy()).cuda() for i in range(len(specs))] for r in range(n)]
            E.esp_sync_many_loopback(ws, ctxs, dev)
            torch.cuda.synchronize()
            for w in ws:
                w.check()
            for i, (k, ro, p, N) in enumerate(specs):
                for r in range(n):
                    where = f"n={n} g={g} {k}/{ro}/p{p} N={N} step={s} rank={r}"
                    got = dev[r][i].cpu().numpy()
                    if k in O.QUANTIZED:
                        np.testing.assert_allclose(got, refs[i].outs[r], rtol=1e-6, atol=1e-30, err_msg=where)
                    else:
                        bad = np.nonzero(bits(got) != bits(refs[i].outs[r]))[0]
                        assert bad.size == 0, f"{where}: {bad.size} mismatches at {bad[:5]}"
                        if sts[i][r].r.size == 0:
                            continue   # empty shard: no state
                        _, rg, _ = ctxs[r][i].get_state()
                        assert np.array_equal(bits(rg[0]), bits(sts[i][r].r)), where + " shard residual"
    finally:
        for w in ws:
            w.destroy()


CASES = [("dgc", "allgather", 0), ("dgc", "alltoall_allgather", 0), ("dgc", "alltoall_allgather", 2),
         ("randomk", "gather_broadcast", 0), ("topk", "allgather", 0), ("efsignsgd", "alltoall_allgather", 0),
         ("onebit", "allgather", 0), ("efsignsgd", "gather_broadcast", 0)]


@pytest.mark.parametrize("n,g", [(8, 4), (4, 2), (6, 3), (8, 2)])
@pytest.mark.parametrize("kind,routine,process", CASES)
def test_hier_loopback(n, g, kind, routine, process):
    run(n, g, [(kind, routine, process, 20_011)])


@pytest.mark.parametrize("n,g", [(8, 4), (4, 4), (4, 1)])
def test_hier_loopback_mixed(n, g):
    """Several tensors (sizes with empty shards, both processes) in one call:
    one machine (g = n: the inter phase is a single rank's identity routine)
    and one GPU per machine (g = 1: the flat routine)."""
    specs = [("dgc", "allgather", 0, 70_001), ("efsignsgd", "alltoall_allgather", 0, 9000),
             ("dgc", "gather_broadcast", 2, 33), ("randomk", "allgather", 0, 4096),
             ("onebit", "alltoall_allgather", 1, 100)]
    run(n, g, specs, steps=3, ratio=0.01)
