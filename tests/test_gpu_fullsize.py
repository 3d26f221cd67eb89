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
