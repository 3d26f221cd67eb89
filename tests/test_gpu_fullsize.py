"""Parity at BASELINE.json's full size in the launch configuration bench.py
times (config 4: BERT-large, 398 tensors, 336,226,108 params, DGC top-0.1%,
Allgather, one bucket, NCCL world).

Every tensor is checked with properties that pin the exact result at any size
(O(N) numpy, no sort): exactly k selected; every selected key exceeds every
unselected key, and among keys equal to the k-th the selected ones are the
lowest indices (the (key desc, idx asc) order of reading R2); the EF identity
out + r_new == acc bit for bit with out * r_new == 0.  Sampled tensors (the
largest, a mid-size one, a 1024-element one) are compared with the oracle
element by element."""
import numpy as np
import pytest

from oracle import esp_oracle as O
from synth import shapes
from synth.values import gradient

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def keys(x):
    return x.view(np.uint32) & np.uint32(0x7FFFFFFF)


def check_topk_exact(acc, sel_mask, k, where):
    assert int(sel_mask.sum()) == k, f"{where}: {int(sel_mask.sum())} selected, k={k}"
    kk = keys(acc)
    T = kk[sel_mask].min()
    un = kk[~sel_mask]
    assert un.size == 0 or un.max() <= T, f"{where}: unselected key above the k-th"
    ties = np.nonzero(kk == T)[0]
    sel_ties = np.nonzero(sel_mask & (kk == T))[0]
    assert np.array_equal(sel_ties, ties[:sel_ties.size]), f"{where}: ties not broken by lowest index"


def test_bert_large_dgc_fullsize():
    assert torch.cuda.is_available()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2205_14465_b200 import esp as E
    torch.cuda.set_device(0)
    sizes = shapes.numels("bert_large")
    ratio = 0.001
    w = E.World.nccl_single(0)
    try:
        ctxs = [E.Ctx(w, "dgc", "allgather", N, tensor_id=t, ratio=ratio) for t, N in enumerate(sizes)]
        grads = [gradient(N, tensor=t) for t, N in enumerate(sizes)]
        dev = [torch.from_numpy(g).cuda() for g in grads]
        E.esp_sync_many(w, ctxs, dev)
        torch.cuda.synchronize()
        sample = {0, int(np.argsort(sizes)[len(sizes) // 2]), sizes.index(1024)}
        for t, N in enumerate(sizes):
            out = dev[t].cpu().numpy()
            _, r, _ = ctxs[t].get_state()
            r = r[0]
            acc = grads[t]                        # step 0: r_old = 0, acc = g + 0 = g (bitwise for g != -0)
            acc = (acc + np.float32(0)).astype(np.float32)
            assert np.array_equal((out + r).view(np.uint32), acc.view(np.uint32)), f"tensor {t}: out + r != acc"
            assert not np.any((out != 0) & (r != 0)), f"tensor {t}: out * r != 0"
            sel = r == 0
            sel &= acc != 0
            check_topk_exact(acc, sel, O.k_of(N, ratio), f"tensor {t} N={N}")
            if t in sample:
                ref = O.sync("allgather", O.Cfg("dgc", ratio), [grads[t]], O.new_states(1, N, "allgather", O.Cfg("dgc", ratio)))
                assert np.array_equal(out.view(np.uint32), ref.outs[0].view(np.uint32)), f"tensor {t} vs oracle"
    finally:
        w.destroy()


def _bench_rule(name):
    import bench
    return bench.workload(name, 1)[1], bench.opt


def test_resnet50_efsignsgd_fullsize():
    """BASELINE config 3 at full size in bench.py's launch configuration:
    ResNet-50's 161 tensors (25,557,032 params), EFSignSGD via Alltoall/
    Allgather (process 2: a7 recompression with the second residual), one
    esp_sync_many over the whole set, two steps (the second lock-stepped from
    the oracle's state).  Every tensor element by element against the oracle
    (1e-6 relative: fp64-reduced scales)."""
    from paper_2205_14465_b200 import esp as E
    torch.cuda.set_device(0)
    sizes = shapes.numels("resnet50")
    w = E.World.nccl_single(0)
    try:
        ctxs = [E.Ctx(w, "efsignsgd", "alltoall_allgather", N, tensor_id=t, ratio=1.0) for t, N in enumerate(sizes)]
        cfg = O.Cfg("efsignsgd", 1.0)
        sts = [O.new_states(1, N, "alltoall_allgather", cfg) for N in sizes]
        for s in range(2):
            if s:
                for t in range(len(sizes)):
                    r2 = np.zeros((1, ctxs[t].get_state()[2].shape[1]), np.float32)
                    r2[0, :sts[t][0].r2.size] = sts[t][0].r2
                    ctxs[t].set_state(sts[t][0].step, sts[t][0].r[None], r2)
            grads = [gradient(N, step=s, tensor=t) for t, N in enumerate(sizes)]
            dev = [torch.from_numpy(g).cuda() for g in grads]
            E.esp_sync_many(w, ctxs, dev)
            torch.cuda.synchronize()
            for t, N in enumerate(sizes):
                ref = O.sync("alltoall_allgather", cfg, [grads[t]], sts[t], tensor_id=t)
                np.testing.assert_allclose(dev[t].cpu().numpy(), ref.outs[0], rtol=1e-6, atol=1e-30,
                                           err_msg=f"resnet50 tensor {t} N={N} step {s}")
    finally:
        w.destroy()


def test_gpt2_medium_mixed_fullsize():
    """BASELINE config 5 at full size in bench.py's launch configuration: GPT-2
    medium's 292 tensors (354,823,168 params) under bench.py's fixed rule --
    DGC 1% Allgather for N >= 2^22 (49 tensors, incl. the 51,463,168-element
    embedding, k = 514,632), EFSignSGD Alltoall/Allgather for 2^20 <= N < 2^22,
    NONE Allreduce below -- in one esp_sync_many.  DGC tensors: the O(N)
    exact-top-k and EF-identity checks; sign tensors element by element
    against the oracle (1e-6 relative); NONE: the identity at n = 1."""
    from paper_2205_14465_b200 import esp as E
    torch.cuda.set_device(0)
    rule, opt = _bench_rule("gpt2_medium_mixed")
    sizes = shapes.numels("gpt2_medium")
    w = E.World.nccl_single(0)
    try:
        opts = [opt(rule, N) for N in sizes]
        ctxs = [E.Ctx(w, k, ro, N, tensor_id=t, ratio=ra, **ex) for t, (N, (k, ra, ro, ex)) in enumerate(zip(sizes, opts))]
        grads = [gradient(N, tensor=t) for t, N in enumerate(sizes)]
        dev = [torch.from_numpy(g).cuda() for g in grads]
        E.esp_sync_many(w, ctxs, dev)
        torch.cuda.synchronize()
        seen = set()
        for t, (N, (k, ra, ro, ex)) in enumerate(zip(sizes, opts)):
            seen.add(k)
            out = dev[t].cpu().numpy()
            where = f"gpt2 tensor {t} N={N} {k}/{ro}"
            if k == "dgc":
                _, r, _ = ctxs[t].get_state()
                r = r[0]
                acc = (grads[t] + np.float32(0)).astype(np.float32)
                assert np.array_equal((out + r).view(np.uint32), acc.view(np.uint32)), where + ": out + r != acc"
                assert not np.any((out != 0) & (r != 0)), where + ": out * r != 0"
                check_topk_exact(acc, (r == 0) & (acc != 0), O.k_of(N, ra), where)
            elif k == "efsignsgd":
                cfg = O.Cfg(k, ra)
                ref = O.sync(ro, cfg, [grads[t]], O.new_states(1, N, ro, cfg), tensor_id=t)
                np.testing.assert_allclose(out, ref.outs[0], rtol=1e-6, atol=1e-30, err_msg=where)
            else:
                assert np.array_equal(out.view(np.uint32), grads[t].view(np.uint32)), where
        assert seen == {"dgc", "efsignsgd", "none"}
    finally:
        w.destroy()
