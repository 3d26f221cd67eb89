"""One rank of the multi-process (NCCL world) parity run, launched by
tests/test_gpu_nccl.py through torch.distributed.run (one process per GPU).

Every rank regenerates all n ranks' seeded gradients, runs the oracle's n-rank
simulation on the host, and compares its OWN CUDA output and EF state with the
oracle's entry for its rank — no result ever travels from the CUDA path to the
oracle.  Byte-moving routines are bit-exact; NCCL-reduced ones (Allreduce,
Reduce-scatter/Allgather, Reduce/Broadcast) are checked against the fp64 mean
within 1e-6 * mean|x| (NCCL's summation order is opaque)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import esp_oracle as O  # noqa: E402
from paper_2205_14465_b200 import esp as E  # noqa: E402
from synth.values import gradient  # noqa: E402

REDUCED = ("allreduce", "reducescatter_allgather", "reduce_broadcast")


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def check(kind, routine, got, ref, grads_all, where):
    if routine in REDUCED:
        x = np.stack([g.astype(np.float64) for g in grads_all])
        scale = np.abs(x).mean(0)
        if kind == "none":
            exact = x.mean(0)
        else:
            exact = ref.astype(np.float64)
            scale = np.maximum(scale, np.abs(exact))
        err = np.abs(got.astype(np.float64) - exact)
        assert np.all(err <= 1e-6 * scale + 1e-30), f"{where}: max err {err.max()}"
    elif kind in O.QUANTIZED:
        np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-30, err_msg=where)
    else:
        bad = np.nonzero(bits(got) != bits(ref))[0]
        assert bad.size == 0, f"{where}: {bad.size} mismatches at {bad[:5]}"


def main():
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = E.World.nccl(local)
    pairs = [(k, r, 0, True) for k in O.KINDS for r in O.ROUTINES if O.legal(O.Cfg(k), r)]
    # the other process of each divisible routine (R19)
    pairs += [(k, r, 2 if k in O.SPARSE else 1, True) for k in ("dgc", "randomk", "efsignsgd")
              for r in ("alltoall_allgather", "gather_broadcast")]
    # Randomk with per-rank indices (R5) through the fused routines
    pairs += [("randomk", r, p, False) for r, p in (("allgather", 0), ("alltoall_allgather", 1),
                                                   ("alltoall_allgather", 2), ("gather_broadcast", 2))]
    N = 30_011
    checked = 0
    for t, (kind, routine, proc, shared) in enumerate(pairs):
        if os.environ.get("ESP_TEST_VERBOSE"):
            print(f"rank {rank}: {kind}/{routine}/process {proc}", flush=True)
        ctx = E.Ctx(w, kind, routine, N, tensor_id=t, ratio=0.02, process=proc, shared_indices=shared)
        cfg = O.Cfg(kind, 0.02, shared_indices=shared, process=proc)
        st = O.new_states(n, N, routine, cfg)
        for s in range(3):
            if kind in O.QUANTIZED and s > 0:   # lock-step: oracle state -> GPU
                r2 = np.zeros((1, ctx.get_state()[2].shape[1]), np.float32)
                if st[rank].r2 is not None:
                    r2[0, :st[rank].r2.size] = st[rank].r2
                ctx.set_state(st[rank].step, st[rank].r[None], r2)
            grads = [gradient(N, step=s, rank=r, tensor=t) for r in range(n)]
            ref = O.sync(routine, cfg, grads, st, tensor_id=t)
            g = torch.from_numpy(grads[rank].copy()).cuda()
            E.esp_sync(w, ctx, g)
            torch.cuda.synchronize()
            check(kind, routine, g.cpu().numpy(), ref.outs[rank], grads, f"rank {rank} {kind}/{routine} step {s}")
            if kind != "none" and routine not in REDUCED:
                _, rg, _ = ctx.get_state()
                if kind in O.QUANTIZED:
                    np.testing.assert_allclose(rg[0], st[rank].r, rtol=1e-6, atol=1e-30)
                else:
                    assert np.array_equal(bits(rg[0]), bits(st[rank].r)), f"residual {kind}/{routine}"
                    if st[rank].r2 is not None:
                        _, _, r2g = ctx.get_state()
                        assert np.array_equal(bits(r2g[0, :st[rank].r2.size]), bits(st[rank].r2)), "r2"
            checked += 1
        c = w.counters()
        w.reset_counters()
        exp = ref.counters[rank]
        assert c["recv"] == 3 * exp.recv and c["sent"] == 3 * exp.sent, (kind, routine, c["recv"], exp.recv)
        ctx.destroy()

    # a mixed strategy through esp_sync_many (bucketing + pipelining with small buckets)
    # a mixed strategy through esp_sync_many (bucketing + pipelining with small
    # buckets), including tensors smaller than n x 32 (empty partitions), both
    # processes and momentum, for 3 steps (EF carried across calls and both
    # call parities of the fused buffers)
    specs = [("dgc", "allgather", 70_000, {}), ("none", "allreduce", 1000, {}),
             ("efsignsgd", "alltoall_allgather", 9000, {}), ("dgc", "alltoall_allgather", 40_000, {}),
             ("onebit", "gather_broadcast", 5000, {}), ("dgc", "allgather", 33, {}),
             ("efsignsgd", "alltoall_allgather", 40, {}), ("dgc", "alltoall_allgather", 50, {"process": 2}),
             ("randomk", "alltoall_allgather", 3000, {"process": 2}), ("topk", "gather_broadcast", 77, {"process": 2}),
             ("dgc", "allgather", 12_345, {"momentum": 0.9}), ("efsignsgd", "alltoall_allgather", 6000, {"process": 1})]
    w.set_bucket_elems(50_000)
    ctxs = [E.Ctx(w, k, r, N_, tensor_id=100 + i, ratio=0.01, **ex) for i, (k, r, N_, ex) in enumerate(specs)]
    cfgs = [O.Cfg(k, 0.01, **ex) for (k, r, N_, ex) in specs]
    sts = [O.new_states(n, N_, r, cfgs[i]) for i, (k, r, N_, _) in enumerate(specs)]
    for s in range(3):
        for i, (k, r, N_, _) in enumerate(specs):
            if k in O.QUANTIZED and s > 0:   # lock-step: oracle state -> GPU
                r2 = np.zeros((1, ctxs[i].get_state()[2].shape[1]), np.float32)
                if sts[i][rank].r2 is not None:
                    r2[0, :sts[i][rank].r2.size] = sts[i][rank].r2
                ctxs[i].set_state(sts[i][rank].step, sts[i][rank].r[None], r2)
        grads = [[gradient(N_, step=s, rank=q, tensor=100 + i) for q in range(n)] for i, (_, _, N_, _) in enumerate(specs)]
        refs = [O.sync(r, cfgs[i], grads[i], sts[i], tensor_id=100 + i) for i, (k, r, _, _) in enumerate(specs)]
        gs = [torch.from_numpy(grads[i][rank].copy()).cuda() for i in range(len(specs))]
        E.esp_sync_many(w, ctxs, gs)
        torch.cuda.synchronize()
        for i, (k, r, _, _) in enumerate(specs):
            check(k, r, gs[i].cpu().numpy(), refs[i].outs[rank], grads[i], f"sync_many {k}/{r} step {s}")
    # back to back: T calls with no host synchronisation between them and a
    # rank-dependent GPU delay before some, so fast ranks run ahead into the
    # next call (both parities of the fused buffers and arrival counters
    # reused while a slow peer is still pushing the previous call)
    w.set_bucket_elems(0)
    bspecs = [("dgc", "allgather", 20_000, {}), ("dgc", "alltoall_allgather", 30_000, {}),
              ("dgc", "alltoall_allgather", 9000, {"process": 2}), ("randomk", "gather_broadcast", 7000, {}),
              ("topk", "gather_broadcast", 5000, {}), ("none", "allreduce", 3000, {}),
              ("randomk", "allgather", 4000, {"shared_indices": False})]
    T = 6
    bctx = [E.Ctx(w, k, r, N_, tensor_id=300 + i, ratio=0.01, **ex) for i, (k, r, N_, ex) in enumerate(bspecs)]
    bcfg = [O.Cfg(k, 0.01, **ex) for (k, r, N_, ex) in bspecs]
    bst = [O.new_states(n, N_, r, bcfg[i]) for i, (k, r, N_, _) in enumerate(bspecs)]
    ball = [[[gradient(N_, step=s, rank=q, tensor=300 + i) for q in range(n)] for i, (_, _, N_, _) in enumerate(bspecs)]
            for s in range(T)]
    bg = [[torch.from_numpy(ball[s][i][rank].copy()).cuda() for i in range(len(bspecs))] for s in range(T)]
    torch.cuda.synchronize()
    dist.barrier()
    for s in range(T):
        if (s + rank) % 2 == 1:
            torch.cuda._sleep(2_000_000 * (1 + rank))   # ~1-4 ms of skew on this rank
        E.esp_sync_many(w, bctx, bg[s])
    torch.cuda.synchronize()
    for s in range(T):
        for i, (k, r, _, _) in enumerate(bspecs):
            ref = O.sync(r, bcfg[i], ball[s][i], bst[i], tensor_id=300 + i)
            check(k, r, bg[s][i].cpu().numpy(), ref.outs[rank], ball[s][i], f"back-to-back {k}/{r} step {s}")
    w.check()
    w.destroy()

    if n > 1:
        multicast_allgather(rank, local, n)
        hierarchical(rank, local, n)
        missing_peer(rank, local)
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}: {checked} pair-steps + sync_many ok", flush=True)


def multicast_allgather(rank, local, n):
    """NVLS multicast forced on (esp_world_set_multicast(1); unicast peer copies
    wherever a GPU lacks it): every Allgather compressor in one esp_sync_many,
    4 back-to-back steps (both call parities twice), bit-exact against the
    oracle; with multicast a rank stores its slot once ("pushed" = the slot,
    not (n-1) slots)."""
    w = E.World.nccl(local)
    w.set_multicast(1)
    specs = [("dgc", 40_000, {}), ("topk", 3000, {}), ("randomk", 20_000, {"shared_indices": False}),
             ("efsignsgd", 9000, {}), ("onebit", 5000, {}), ("dgc", 77, {"approx": True})]
    ctxs = [E.Ctx(w, k, "allgather", N_, tensor_id=500 + i, ratio=0.01, **ex) for i, (k, N_, ex) in enumerate(specs)]
    cfgs = [O.Cfg(k, 0.01, shared_indices=ex.get("shared_indices", True), approx=ex.get("approx", False))
            for (k, N_, ex) in specs]
    sts = [O.new_states(n, N_, "allgather", cfgs[i]) for i, (k, N_, _) in enumerate(specs)]
    T = 4
    allg = [[[gradient(N_, step=s, rank=q, tensor=500 + i) for q in range(n)] for i, (_, N_, _) in enumerate(specs)]
            for s in range(T)]
    dev = [[torch.from_numpy(allg[s][i][rank].copy()).cuda() for i in range(len(specs))] for s in range(T)]
    torch.cuda.synchronize()
    w.reset_counters()
    for s in range(T):
        for i, (k, _, _) in enumerate(specs):
            if k in O.QUANTIZED and s > 0:   # lock-step from the oracle (after the previous call completed)
                torch.cuda.synchronize()
                ctxs[i].set_state(sts[i][rank].step, sts[i][rank].r[None])
        E.esp_sync_many(w, ctxs, dev[s])
        torch.cuda.synchronize()
        for i, (k, _, _) in enumerate(specs):
            ref = O.sync("allgather", cfgs[i], allg[s][i], sts[i], tensor_id=500 + i)
            check(k, "allgather", dev[s][i].cpu().numpy(), ref.outs[rank], allg[s][i], f"multicast {k} step {s}")
    c = w.counters()
    slot = sum(x.payload_bytes for x in ctxs)
    print(f"rank {rank}: multicast allgather ok, pushed {c['pushed'] / T:.0f} B/step, slot ~{slot} B", flush=True)
    w.check()
    w.destroy()


def hierarchical(rank, local, n):
    """Hierarchical sync on real ranks (esp_world_create_hier over NCCL, CUDA
    IPC inside each machine): machines of 2 GPUs (n = 2: one machine; n = 4:
    2 x 2), DGC / EFSignSGD / Randomk, 3 steps, against the oracle."""
    flat = E.World.nccl(local)
    hw = flat.hier(2)
    specs = [("dgc", "allgather", 0, 30_011), ("efsignsgd", "alltoall_allgather", 0, 9000),
             ("randomk", "gather_broadcast", 0, 5000), ("dgc", "alltoall_allgather", 2, 70)]
    ctxs = [E.Ctx(hw, k, ro, N_, tensor_id=600 + i, ratio=0.02, process=p) for i, (k, ro, p, N_) in enumerate(specs)]
    cfgs = [O.Cfg(k, 0.02, process=p) for (k, ro, p, N_) in specs]
    sts = [O.new_states_hier(n, N_, ro, cfgs[i], 2) for i, (k, ro, p, N_) in enumerate(specs)]
    for s in range(3):
        for i, (k, ro, p, N_) in enumerate(specs):
            if k in O.QUANTIZED and s > 0:
                st = sts[i][rank]
                r2len = ctxs[i].get_state()[2].shape[1]
                r2 = np.zeros((1, r2len), np.float32)
                if st.r2 is not None:
                    r2[0, :st.r2.size] = st.r2
                ctxs[i].set_state(st.step, st.r[None], r2)
        grads = [[gradient(N_, step=s, rank=q, tensor=600 + i) for q in range(n)] for i, (_, _, _, N_) in enumerate(specs)]
        refs = [O.sync_hierarchical(ro, cfgs[i], grads[i], sts[i], 2, tensor_id=600 + i)
                for i, (k, ro, p, N_) in enumerate(specs)]
        gs = [torch.from_numpy(grads[i][rank].copy()).cuda() for i in range(len(specs))]
        E.esp_sync_many(hw, ctxs, gs)
        torch.cuda.synchronize()
        for i, (k, ro, _, _) in enumerate(specs):
            check(k, ro, gs[i].cpu().numpy(), refs[i].outs[rank], grads[i], f"hierarchical {k}/{ro} step {s}")
    hw.check()
    hw.destroy()
    flat.destroy()
    print(f"rank {rank}: hierarchical ok", flush=True)


def missing_peer(rank, local):
    """A peer that never arrives: rank 0 calls once more than the others; its
    wait gives up after the timeout instead of hanging or trapping, and the
    world reports the failure (the CUDA context stays usable)."""
    w2 = E.World.nccl(local)
    w2.set_timeout(2.0)
    c2 = E.Ctx(w2, "dgc", "allgather", 5000, tensor_id=400, ratio=0.01)
    g2 = torch.from_numpy(gradient(5000, rank=rank, tensor=400)).cuda()
    E.esp_sync(w2, c2, g2)
    torch.cuda.synchronize()
    w2.check()
    dist.barrier()
    if rank == 0:
        E.esp_sync(w2, c2, g2)
        torch.cuda.synchronize()
        try:
            w2.check()
            raise AssertionError("a missing peer was not reported")
        except E.EspError as e:
            assert "did not arrive" in str(e), str(e)
        torch.ones(1, device="cuda").sum().item()   # the context still works
    dist.barrier()
    c2.destroy()
    w2.destroy()


if __name__ == "__main__":
    main()
