"""Parity of the CUDA path (through the C ABI) against the oracle, sim world:
n virtual ranks on one GPU (SURVEY.md 4 layers 2-3).  Bit-exact on indices,
values, packed sign bits, residuals and aggregated outputs wherever the
arithmetic is fixed; fp64-reduced scales within 1e-6 relative (north_star)."""
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


def esp():
    from paper_2205_14465_b200 import esp as E
    return E


def bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def upload(arrs):
    return torch.from_numpy(np.concatenate(arrs)).cuda()


def check_out(kind, got, ref, where):
    if kind in ("dgc", "topk", "randomk", "none"):
        bad = np.nonzero(bits(got) != bits(ref))[0]
        assert bad.size == 0, f"{where}: {bad.size} mismatches, first {bad[:5]} got {got[bad[:5]]} ref {ref[bad[:5]]}"
    else:
        np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-30, err_msg=where)


def run_sim(kind, routine, n, N, steps=3, ratio=0.01, dist="D1", mode="mixed", ef=True,
            reduce="mean", shared=True, lockstep=None, tensor_id=3, seed=11, process=0, approx=False,
            sample_rate=0.0):
    """Run `steps` syncs in a sim world and compare every rank's output and
    residual with the oracle after each step."""
    E = esp()
    if lockstep is None:
        lockstep = kind in O.QUANTIZED
    w = E.World.sim(n, 0)
    ctx = E.Ctx(w, kind, routine, N, tensor_id=tensor_id, ratio=ratio, error_feedback=ef, seed=seed,
                shared_indices=shared, reduce=reduce, process=process, approx=approx, sample_rate=sample_rate)
    cfg = O.Cfg(kind, ratio, ef, seed, shared, reduce, process, approx=approx, sample_rate=sample_rate)
    st = O.new_states(n, N, routine, cfg)
    try:
        for s in range(steps):
            if lockstep and s > 0:
                # oracle -> GPU: re-seed the GPU state from the oracle's (never the reverse)
                r = np.stack([x.r for x in st])
                r2len = ctx.get_state()[2].shape[1]
                r2 = np.zeros((n, r2len), np.float32)
                for i, x in enumerate(st):
                    if x.r2 is not None:
                        r2[i, :x.r2.size] = x.r2
                ctx.set_state(st[0].step, r, r2)
            grads = [gradient(N, step=s, rank=r, tensor=tensor_id, dist=dist, mode=mode) for r in range(n)]
            ref = O.sync(routine, cfg, grads, st, tensor_id=tensor_id)
            g = upload(grads)
            E.esp_sync(w, ctx, g)
            torch.cuda.synchronize()
            out = g.cpu().numpy().reshape(n, N)
            for r in range(n):
                check_out(kind, out[r], ref.outs[r], f"{kind}/{routine} n={n} N={N} step={s} rank={r} out")
            if kind != "none":
                step, rg, r2g = ctx.get_state()
                assert step == st[0].step
                for r in range(n):
                    if kind in O.QUANTIZED:
                        np.testing.assert_allclose(rg[r], st[r].r, rtol=1e-6, atol=1e-30)
                    else:
                        assert np.array_equal(bits(rg[r]), bits(st[r].r)), f"residual rank {r} step {s}"
                    if st[r].r2 is not None and kind in O.QUANTIZED:
                        np.testing.assert_allclose(r2g[r, :st[r].r2.size], st[r].r2, rtol=1e-6, atol=1e-30)
                    elif st[r].r2 is not None:   # sparse second residual: exact
                        assert np.array_equal(bits(r2g[r, :st[r].r2.size]), bits(st[r].r2)), f"r2 rank {r} step {s}"
        return w
    finally:
        w.destroy()


# DGC / TOPK h1 has two paths: buckets that fit the chip's shared memory run the
# one-kernel on-chip select (dgc_mid_kernel), larger ones the sample / stream /
# finalize chain; ESP_DGC_PATH=chain (read when a plan is built) forces the
# chain so that both stay covered at every size
PATHS = ["onchip", "chain"]


def set_path(monkeypatch, path):
    if path == "chain":
        monkeypatch.setenv("ESP_DGC_PATH", "chain")
    else:
        monkeypatch.delenv("ESP_DGC_PATH", raising=False)


# ---------------------------------------------------------------- config 1
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("N", [1 << 20, 10 ** 6])
def test_config1_dgc_allgather_n2(N, path, monkeypatch):
    """BASELINE config 1: 1M-element fp32 gradient, DGC top-1% with EF, Allgather,
    n = 2 simulated ranks, 5 steps, bit-exact."""
    set_path(monkeypatch, path)
    run_sim("dgc", "allgather", 2, N, steps=5, ratio=0.01)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("dist", ["D1", "D2", "D3"])
@pytest.mark.parametrize("N", [1, 31, 33, 1000, 4097, 8193, (1 << 16) + 3, 100_003])
def test_dgc_sizes_dists(N, dist, path, monkeypatch):
    set_path(monkeypatch, path)
    run_sim("dgc", "allgather", 2, N, steps=2, ratio=0.01, dist=dist)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("mode", ["equal", "zeros", "spike", "pm0", "denormal", "mixed"])
def test_dgc_adversarial(mode, path, monkeypatch):
    # all-equal magnitudes force the fallback and the tie-break; zeros give T = 0
    set_path(monkeypatch, path)
    run_sim("dgc", "allgather", 2, 50_001, steps=2, ratio=0.01, dist="D4", mode=mode)


@pytest.mark.parametrize("force", ["1", "3"])
@pytest.mark.parametrize("N", [3000, 50_001, 600_001])
def test_dgc_forced_fallback(force, N, monkeypatch):
    """The sampled threshold only accelerates: forcing every segment through the
    fallback (1: recompaction at thr_lo; 3: thr_lo misses too -> thr = 0) must
    leave the selection bit-identical (reading R3)."""
    monkeypatch.setenv("ESP_DGC_FORCE_FALLBACK", force)
    set_path(monkeypatch, "chain")   # the on-chip select has no sampled threshold
    run_sim("dgc", "allgather", 2, N, steps=2, ratio=0.01)
    run_sim("dgc", "alltoall_allgather", 4, N, steps=2, ratio=0.01)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("ratio", [0.001, 0.05, 0.5, 1.0])
def test_dgc_ratios(ratio, path, monkeypatch):
    set_path(monkeypatch, path)
    run_sim("dgc", "allgather", 2, 70_000, steps=2, ratio=ratio)


# ---------------------------------------------------------------- every pair
PAIRS = [(k, r) for k in O.KINDS for r in O.ROUTINES if O.legal(O.Cfg(k), r)]


@pytest.mark.parametrize("kind,routine", PAIRS)
@pytest.mark.parametrize("n", [2, 4, 8])
def test_pairs_sim(kind, routine, n):
    run_sim(kind, routine, n, 20_011, steps=3, ratio=0.02)


@pytest.mark.parametrize("kind", ["efsignsgd", "onebit"])
@pytest.mark.parametrize("N", [1, 32, 33, 1023, 8193, 300_007])
def test_sign_sizes(kind, N):
    run_sim(kind, "allgather", 2, N, steps=2)
    run_sim(kind, "alltoall_allgather", 4, N, steps=2)


@pytest.mark.parametrize("kind", ["efsignsgd", "onebit"])
@pytest.mark.parametrize("routine,process", [("allgather", 0), ("alltoall_allgather", 2), ("alltoall_allgather", 1),
                                             ("gather_broadcast", 2)])
def test_sign_segments_beyond_one_finalize_chunk(kind, routine, process):
    """Segments longer than kFinRuns x 512 = 8,388,608 elements take the
    finalize kernel's two-level (chunked) reduction of the per-run partials,
    in h1 and in a7 -- the path config 2's 2^26..2^30-byte sweep points and
    large tensors run.  N = 2^24 + 2^20 + 77: whole-tensor segments of 17.8 M
    elements, Alltoall partitions of 8.9 M (n = 2)."""
    run_sim(kind, routine, 2, (1 << 24) + (1 << 20) + 77, steps=2, process=process)


# ---------------------------------------------- DGC approximate-count mode (R22, NEXT-2)
@pytest.mark.parametrize("N,ratio,rate", [(1000, 0.01, 0.0), (50_001, 0.01, 0.0), (1 << 20, 0.01, 0.0),
                                          (1 << 20, 0.001, 0.0), (300_007, 0.01, 0.005), (2_000_003, 0.001, 0.0005)])
@pytest.mark.parametrize("routine,process", [("allgather", 0), ("alltoall_allgather", 1),
                                             ("alltoall_allgather", 2), ("gather_broadcast", 2)])
def test_dgc_approx_mode(N, ratio, rate, routine, process):
    """The sampled threshold decides the result here, so the GPU sampler (hashed
    strata, the round(rho s)-th sampled key's 21-bit prefix) must match the
    oracle's bit for bit; fewer than k entries are padded.  Bit-exact outputs
    and residuals over 3 steps (EF carried)."""
    run_sim("dgc", routine, 2, N, steps=3, ratio=ratio, process=process, approx=True, sample_rate=rate)


def test_dgc_approx_more_ranks_and_exact_rate():
    run_sim("dgc", "allgather", 8, 200_003, steps=3, ratio=0.01, approx=True)
    run_sim("dgc", "alltoall_allgather", 4, 200_003, steps=2, ratio=0.01, sample_rate=0.003)   # exact, other sampler


def test_randomk_unshared_and_sum():
    run_sim("randomk", "allgather", 4, 10_000, steps=3, ratio=0.03, shared=False)
    run_sim("dgc", "allgather", 4, 10_000, steps=2, reduce="sum")
    run_sim("efsignsgd", "gather_broadcast", 4, 10_000, steps=2, reduce="sum")


def test_no_error_feedback():
    for kind in ("dgc", "randomk", "efsignsgd", "onebit"):
        run_sim(kind, "allgather", 2, 9_999, steps=2, ef=False)


def test_n1_world():
    for kind, routine in PAIRS:
        run_sim(kind, routine, 1, 5_000, steps=2, ratio=0.05)


# ---------------------------------------------------------------- h1 / h2 ABI
@pytest.mark.parametrize("kind", ["dgc", "randomk", "efsignsgd", "onebit"])
def test_compress_payload_bytes(kind):
    """esp_compress payload == the oracle's serialized chunks (sparse: byte for
    byte; sign: words byte for byte, scale header within 1e-6)."""
    E = esp()
    n, N = 2, 33_333
    w = E.World.sim(n, 0)
    try:
        ctx = E.Ctx(w, kind, "alltoall_allgather", N, tensor_id=5, ratio=0.01)
        cfg = O.Cfg(kind, 0.01)
        st = O.new_states(n, N, "alltoall_allgather", cfg)
        grads = [gradient(N, rank=r, tensor=5) for r in range(n)]
        ref = O.sync("alltoall_allgather", cfg, grads, st, tensor_id=5)
        pay = E.esp_compress(ctx, upload(grads))
        torch.cuda.synchronize()
        pay = pay.cpu().numpy().reshape(n, -1)
        assert pay.shape[1] == len(ref.payloads[0])
        cb = O.chunk_bytes(cfg, N, n)
        for r in range(n):
            got, exp = pay[r].tobytes(), ref.payloads[r]
            for p in range(n):
                gc, ec = got[p * cb:(p + 1) * cb], exp[p * cb:(p + 1) * cb]
                if kind in O.SPARSE:
                    assert gc == ec, f"rank {r} chunk {p}"
                else:
                    assert gc[16:] == ec[16:], f"words rank {r} chunk {p}"
                    np.testing.assert_allclose(np.frombuffer(gc[:8], np.float32),
                                               np.frombuffer(ec[:8], np.float32), rtol=1e-6)
        # h2 through esp_decompress == oracle aggregation of the same pieces
        pieces = [torch.from_numpy(pay[r].copy()).cuda() for r in range(n)]
        out = torch.empty(N, dtype=torch.float32, device="cuda")
        E.esp_decompress(ctx, pieces, out)
        torch.cuda.synchronize()
        if kind in O.SPARSE:
            check_out(kind, out.cpu().numpy(), ref.outs[0], "decompress")
    finally:
        w.destroy()


@pytest.mark.parametrize("kind", ["dgc", "randomk", "efsignsgd", "onebit"])
def test_decompress_accumulate(kind):
    """esp_decompress(..., accumulate=1): out[i] := fl(out[i] + agg[i]) for every
    i, agg = the rank-order mean of the pieces' decodes.  The
    three pieces are fresh-state compressions of three gradients (one ctx each,
    the same tensor id), so the oracle's compress_segment of each gradient is
    the exact payload."""
    E = esp()
    N = 50_003
    w = E.World.nccl_single(0)
    try:
        grads = [gradient(N, rank=r, tensor=4) for r in range(3)]
        cfg = O.Cfg(kind, 0.02)
        ctxs = [E.Ctx(w, kind, "allgather", N, tensor_id=4, ratio=0.02) for _ in range(3)]
        pays = [E.esp_compress(c, torch.from_numpy(g.copy()).cuda()) for c, g in zip(ctxs, grads)]
        dec = [O.compress_segment(cfg, g, tensor_id=4)[1] for g in grads]
        agg = O.aggregate(dec, "mean", 3)
        out0 = gradient(N, rank=9, tensor=5, dist="D2")
        out = torch.from_numpy(out0.copy()).cuda()
        E.esp_decompress(ctxs[0], pays, out, accumulate=True)
        torch.cuda.synchronize()
        want = (out0 + agg).astype(np.float32)
        check_out(kind, out.cpu().numpy(), want, f"accumulate {kind}")
    finally:
        w.destroy()


def test_sync_many_equals_single():
    """A mixed strategy over a tensor set (bucketing, multi-tensor tables, small
    buckets to exercise the pipeline) equals per-tensor oracle syncs."""
    E = esp()
    n = 4
    specs = [("dgc", "allgather", 5000), ("none", "allreduce", 1000), ("efsignsgd", "alltoall_allgather", 7000),
             ("dgc", "allgather", 33), ("randomk", "allreduce", 4000), ("onebit", "gather_broadcast", 3000),
             ("dgc", "alltoall_allgather", 9000), ("none", "reduce_broadcast", 17), ("dgc", "allgather", 70000)]
    w = E.World.sim(n, 0)
    w.set_bucket_elems(20000)
    try:
        ctxs = [E.Ctx(w, k, r, N, tensor_id=t, ratio=0.01) for t, (k, r, N) in enumerate(specs)]
        sts = [O.new_states(n, N, r, O.Cfg(k, 0.01)) for (k, r, N) in specs]
        for s in range(3):
            for t, (k, r, N) in enumerate(specs):
                if k in O.QUANTIZED and s > 0:
                    st = sts[t]
                    r2 = np.zeros((n, ctxs[t].get_state()[2].shape[1]), np.float32)
                    for i, x in enumerate(st):
                        if x.r2 is not None:
                            r2[i, :x.r2.size] = x.r2
                    ctxs[t].set_state(st[0].step, np.stack([x.r for x in st]), r2)
            grads = [[gradient(N, step=s, rank=r, tensor=t) for r in range(n)] for t, (_, _, N) in enumerate(specs)]
            refs = [O.sync(r, O.Cfg(k, 0.01), grads[t], sts[t], tensor_id=t) for t, (k, r, N) in enumerate(specs)]
            gs = [upload(grads[t]) for t in range(len(specs))]
            E.esp_sync_many(w, ctxs, gs)
            torch.cuda.synchronize()
            for t, (k, r, N) in enumerate(specs):
                out = gs[t].cpu().numpy().reshape(n, N)
                for rr in range(n):
                    check_out(k, out[rr], refs[t].outs[rr], f"sync_many t={t} {k}/{r} step {s} rank {rr}")
    finally:
        w.destroy()


def test_counters_match_cost_table():
    """Byte counters of the instrumented comm layer == the oracle's counters ==
    the cost table's closed forms."""
    E = esp()
    n, N = 4, 12_345
    for kind, routine in PAIRS:
        w = E.World.sim(n, 0)
        try:
            ctx = E.Ctx(w, kind, routine, N, ratio=0.01)
            cfg = O.Cfg(kind, 0.01)
            ref = O.sync(routine, cfg, [gradient(N, rank=r) for r in range(n)], O.new_states(n, N, routine, cfg))
            E.esp_sync(w, ctx, upload([gradient(N, rank=r) for r in range(n)]))
            torch.cuda.synchronize()
            for lr in range(n):
                c = w.counters(lr)
                assert c["recv"] == ref.counters[lr].recv, (kind, routine, lr)
                assert c["sent"] == ref.counters[lr].sent, (kind, routine, lr)
            c0 = w.counters(0)
            assert (c0["h1_calls"], c0["h2_pieces"]) == (ref.counters[0].h1, ref.counters[0].h2), (kind, routine)
        finally:
            w.destroy()


# ---------------------------------------------------------------- ABI negative tests
def test_abi_errors():
    E = esp()
    w = E.World.sim(2, 0)
    try:
        with pytest.raises(E.EspError) as ei:
            E.Ctx(w, "dgc", "allreduce", 100)
        assert ei.value.status == 2
        with pytest.raises(E.EspError) as ei:
            E.Ctx(w, "randomk", "allreduce", 100, shared_indices=False)
        assert ei.value.status == 2
        with pytest.raises(E.EspError) as ei:
            E.Ctx(w, "none", "allgather", 100)
        assert ei.value.status == 2
        with pytest.raises(E.EspError) as ei:
            E.Ctx(w, "dgc", "allgather", 1 << 31)
        assert ei.value.status == 3
        with pytest.raises(E.EspError) as ei:
            E.Ctx(w, "dgc", "allgather", 0)
        assert ei.value.status == 1
        with pytest.raises(E.EspError) as ei:
            E.Ctx(w, "dgc", "allgather", 10, ratio=0.0)
        assert ei.value.status == 1
        ctx = E.Ctx(w, "dgc", "allgather", 100)
        g = torch.zeros(201, device="cuda")
        import ctypes
        st_ = E.lib().esp_sync(w.h, ctx.h, ctypes.c_void_p(g.data_ptr() + 2), None)   # not 4-byte aligned
        assert st_ == 1
        w2 = E.World.sim(2, 0)
        try:
            st_ = E.lib().esp_sync(w2.h, ctx.h, ctypes.c_void_p(g.data_ptr()), None)   # ctx of another world
            assert st_ == 7
        finally:
            w2.destroy()
        # the binding rejects what the raw-pointer ABI cannot see
        with pytest.raises(TypeError):
            E.esp_sync(w, ctx, torch.zeros(200, device="cuda", dtype=torch.float16))
        with pytest.raises(ValueError):
            E.esp_sync(w, ctx, torch.zeros(199, device="cuda"))                  # nlocal * numel = 200
        with pytest.raises(ValueError):
            E.esp_sync(w, ctx, torch.zeros(400, device="cuda")[::2])             # not contiguous
        with pytest.raises(ValueError):
            E.esp_sync(w, ctx, torch.zeros(200))                                  # host memory
    finally:
        w.destroy()


# ---------------------------------------------- both processes of both divisible routines
XPROC = [(k, r, p) for k in ("dgc", "topk", "randomk", "efsignsgd", "onebit")
         for r in ("alltoall_allgather", "gather_broadcast") for p in (1, 2)]


@pytest.mark.parametrize("kind,routine,process", XPROC)
@pytest.mark.parametrize("n", [1, 2, 4])
def test_processes(kind, routine, process, n):
    """Process 1 (forward the chunks) and process 2 (decompress, aggregate and
    recompress mid-scheme with r2) of Alltoall/Allgather and Gather/Broadcast
    for every compressor ("the decision tree abstraction covers
    all of them"; R19) against the oracle, 3 steps."""
    run_sim(kind, routine, n, 70_001, steps=3, ratio=0.02, process=process, dist="D3" if kind == "dgc" else "D1")


@pytest.mark.parametrize("process", [1, 2])
def test_processes_unshared_randomk(process):
    run_sim("randomk", "alltoall_allgather", 4, 33_333, steps=2, ratio=0.05, shared=False, process=process)
    run_sim("randomk", "gather_broadcast", 4, 33_333, steps=2, ratio=0.05, shared=False, process=process)


# ---------------------------------------------- DGC momentum correction (R20)
@pytest.mark.parametrize("kind", ["dgc", "topk"])
@pytest.mark.parametrize("routine,n", [("allgather", 2), ("allgather", 4), ("alltoall_allgather", 4),
                                       ("gather_broadcast", 2)])
@pytest.mark.parametrize("path", PATHS)
def test_momentum_correction(kind, routine, n, path, monkeypatch):
    """u = fl(fl(m u) + g), v = fl(v + u), top-k of v, v[sel] = u[sel] = 0:
    outputs, v (the residual) and u bit-exact against the oracle over 4 steps."""
    set_path(monkeypatch, path)
    E = esp()
    N, m = 70_001, 0.9
    w = E.World.sim(n, 0)
    try:
        ctx = E.Ctx(w, kind, routine, N, tensor_id=9, ratio=0.01, momentum=m)
        cfg = O.Cfg(kind, 0.01, momentum=m)
        st = O.new_states(n, N, routine, cfg)
        for s in range(4):
            grads = [gradient(N, step=s, rank=r, tensor=9, dist="D3") for r in range(n)]
            ref = O.sync(routine, cfg, grads, st, tensor_id=9)
            g = upload(grads)
            E.esp_sync(w, ctx, g)
            torch.cuda.synchronize()
            out = g.cpu().numpy().reshape(n, N)
            _, rg, _ = ctx.get_state()
            ug = ctx.get_momentum()
            for r in range(n):
                check_out(kind, out[r], ref.outs[r], f"momentum {kind}/{routine} step {s} rank {r}")
                assert np.array_equal(bits(rg[r]), bits(st[r].r)), f"v rank {r} step {s}"
                assert np.array_equal(bits(ug[r]), bits(st[r].u)), f"u rank {r} step {s}"
    finally:
        w.destroy()


def test_momentum_abi_errors():
    E = esp()
    w = E.World.sim(2, 0)
    try:
        for kw in (dict(kind="randomk"), dict(kind="efsignsgd"), dict(kind="dgc", error_feedback=False)):
            with pytest.raises(E.EspError):
                E.Ctx(w, routine="allgather", numel=100, momentum=0.9, **kw)
        with pytest.raises(E.EspError):
            E.Ctx(w, "dgc", "allgather", 100, momentum=1.0)
        c = E.Ctx(w, "dgc", "allgather", 100)
        with pytest.raises(E.EspError):
            c.get_momentum()
    finally:
        w.destroy()


# ---------------------------------------------- gradients that are only 4-byte aligned
@pytest.mark.parametrize("kind,routine", [(k, r) for k in O.KINDS for r in O.ROUTINES
                                          if O.legal(O.Cfg(k), r)])
def test_unaligned_gradients(kind, routine):
    """esp_sync accepts 4-byte aligned gradients (e.g. the per-parameter views of
    a DDP bucket); the guarded-load paths give the same bits as the oracle."""
    E = esp()
    n, N = 2, 9_999
    w = E.World.sim(n, 0)
    try:
        ctx = E.Ctx(w, kind, routine, N, tensor_id=4, ratio=0.02)
        cfg = O.Cfg(kind, 0.02)
        st = O.new_states(n, N, routine, cfg)
        for s in range(2):
            grads = [gradient(N, step=s, rank=r, tensor=4) for r in range(n)]
            ref = O.sync(routine, cfg, grads, st, tensor_id=4)
            buf = torch.zeros(n * N + 1, device="cuda")
            buf[1:].copy_(upload(grads))
            E.esp_sync(w, ctx, buf[1:])
            torch.cuda.synchronize()
            out = buf[1:].cpu().numpy().reshape(n, N)
            for r in range(n):
                check_out(kind, out[r], ref.outs[r], f"unaligned {kind}/{routine} step {s} rank {r}")
            if kind in O.QUANTIZED:   # lock-step (oracle -> GPU)
                r2len = ctx.get_state()[2].shape[1]
                r2 = np.zeros((n, r2len), np.float32)
                for i, x in enumerate(st):
                    if x.r2 is not None:
                        r2[i, :x.r2.size] = x.r2
                ctx.set_state(st[0].step, np.stack([x.r for x in st]), r2)
    finally:
        w.destroy()


# ---------------------------------- DGC deferred EF zeroing across calls
@pytest.mark.parametrize("kind", ["dgc", "topk"])
@pytest.mark.parametrize("routine,n,process", [("allgather", 2, 0), ("alltoall_allgather", 4, 1),
                                               ("alltoall_allgather", 4, 2), ("gather_broadcast", 2, 2)])
@pytest.mark.parametrize("ratio,momentum", [(0.001, 0.0), (0.01, 0.0), (0.01, 0.9), (0.06, 0.0)])
def test_dgc_deferred_zeroing_multistep(kind, routine, n, process, ratio, momentum, monkeypatch):
    """The write kernel records each call's selection per 4096-element tile
    instead of zeroing r (and u) in memory; the next call's streaming pass
    reads those positions as +0.  Five calls back to back with no state
    read-out in between (get_state would apply the records): every output bit-
    exact against the oracle, then r, r2 and u at the end.  6% overflows the
    64/128-entry records (the rest is zeroed directly); N has a partial tail
    tile; both processes of the divisible routines (process 2: r2's records)."""
    set_path(monkeypatch, "chain")   # the chain's write kernel keeps the records
    E = esp()
    N = 3 * 4096 * 7 + 1234
    w = E.World.sim(n, 0)
    try:
        ctx = E.Ctx(w, kind, routine, N, tensor_id=12, ratio=ratio, momentum=momentum, process=process)
        cfg = O.Cfg(kind, ratio, process=process, momentum=momentum)
        st = O.new_states(n, N, routine, cfg)
        for s in range(5):
            grads = [gradient(N, step=s, rank=r, tensor=12, dist="D2") for r in range(n)]
            ref = O.sync(routine, cfg, grads, st, tensor_id=12)
            g = upload(grads)
            E.esp_sync(w, ctx, g)
            torch.cuda.synchronize()
            out = g.cpu().numpy().reshape(n, N)
            for r in range(n):
                check_out(kind, out[r], ref.outs[r], f"deferred {kind}/{routine} p{process} step {s} rank {r}")
        _, rg, r2g = ctx.get_state()
        for r in range(n):
            assert np.array_equal(bits(rg[r]), bits(st[r].r)), f"residual rank {r}"
            if st[r].r2 is not None:
                assert np.array_equal(bits(r2g[r, :st[r].r2.size]), bits(st[r].r2)), f"r2 rank {r}"
        if momentum:
            ug = ctx.get_momentum()
            for r in range(n):
                assert np.array_equal(bits(ug[r]), bits(st[r].u)), f"u rank {r}"
    finally:
        w.destroy()


def test_dgc_deferred_zeroing_state_roundtrip(monkeypatch):
    """get_state / set_state between calls: reading the state applies the
    pending records (so they are not applied twice), writing it drops them."""
    set_path(monkeypatch, "chain")
    E = esp()
    n, N, ratio = 2, 50_000, 0.01
    w = E.World.sim(n, 0)
    try:
        ctx = E.Ctx(w, "dgc", "allgather", N, tensor_id=13, ratio=ratio)
        cfg = O.Cfg("dgc", ratio)
        st = O.new_states(n, N, "allgather", cfg)
        for s in range(4):
            grads = [gradient(N, step=s, rank=r, tensor=13) for r in range(n)]
            ref = O.sync("allgather", cfg, grads, st, tensor_id=13)
            g = upload(grads)
            E.esp_sync(w, ctx, g)
            torch.cuda.synchronize()
            out = g.cpu().numpy().reshape(n, N)
            for r in range(n):
                check_out("dgc", out[r], ref.outs[r], f"roundtrip step {s} rank {r}")
            if s == 1:   # read-out then write-back of the same state
                step, rg, r2g = ctx.get_state()
                ctx.set_state(step, rg, r2g)
            if s == 2:   # read-out only
                ctx.get_state()
    finally:
        w.destroy()


# ---------------------------------------------- on-chip DGC select (dgc_mid_kernel)
@pytest.mark.parametrize("kind", ["dgc", "topk"])
@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_onchip_after_chain_records(kind, momentum, monkeypatch):
    """Chain calls leave deferred-zeroing records; the on-chip kernel applies
    and clears them before it reads r / u, then zeroes its own selection in
    memory; and back to the chain.  Outputs, r and u bit-exact each step."""
    E = esp()
    n, N, ratio = 2, 5 * 4096 + 77, 0.01
    w = E.World.sim(n, 0)
    try:
        ctx = E.Ctx(w, kind, "allgather", N, tensor_id=21, ratio=ratio, momentum=momentum)
        cfg = O.Cfg(kind, ratio, momentum=momentum)
        st = O.new_states(n, N, "allgather", cfg)
        for s, path in enumerate(["chain", "chain", "onchip", "onchip", "chain", "onchip"]):
            set_path(monkeypatch, path)
            w.drop_plans()
            grads = [gradient(N, step=s, rank=r, tensor=21, dist="D2") for r in range(n)]
            ref = O.sync("allgather", cfg, grads, st, tensor_id=21)
            g = upload(grads)
            E.esp_sync(w, ctx, g)
            torch.cuda.synchronize()
            out = g.cpu().numpy().reshape(n, N)
            for r in range(n):
                check_out(kind, out[r], ref.outs[r], f"{path} step {s} rank {r}")
        _, rg, _ = ctx.get_state()
        for r in range(n):
            assert np.array_equal(bits(rg[r]), bits(st[r].r)), f"residual rank {r}"
        if momentum:
            ug = ctx.get_momentum()
            for r in range(n):
                assert np.array_equal(bits(ug[r]), bits(st[r].u)), f"u rank {r}"
    finally:
        w.destroy()


@pytest.mark.parametrize("path", PATHS)
def test_onchip_many_segments(path, monkeypatch):
    """One DGC bucket of tensors of very different lengths (one tile, several
    CTAs, a ragged tail, an odd length that misaligns the next rank's slice,
    Alltoall partitions): the on-chip kernel maps CTAs to segments from the
    table; every output bit-exact over 3 steps."""
    set_path(monkeypatch, path)
    E = esp()
    n = 4
    specs = [("dgc", "allgather", 4097), ("dgc", "allgather", 300_007), ("dgc", "alltoall_allgather", 123_457),
             ("dgc", "allgather", 64 * 4096), ("topk", "allgather", 50_001), ("dgc", "allgather", 9)]
    w = E.World.sim(n, 0)
    try:
        ctxs = [E.Ctx(w, k, r, N, tensor_id=40 + t, ratio=0.01) for t, (k, r, N) in enumerate(specs)]
        sts = [O.new_states(n, N, r, O.Cfg(k, 0.01)) for (k, r, N) in specs]
        for s in range(3):
            grads = [[gradient(N, step=s, rank=r, tensor=40 + t) for r in range(n)] for t, (_, _, N) in enumerate(specs)]
            refs = [O.sync(r, O.Cfg(k, 0.01), grads[t], sts[t], tensor_id=40 + t) for t, (k, r, N) in enumerate(specs)]
            gs = [upload(grads[t]) for t in range(len(specs))]
            E.esp_sync_many(w, ctxs, gs)
            torch.cuda.synchronize()
            for t, (k, r, N) in enumerate(specs):
                out = gs[t].cpu().numpy().reshape(n, N)
                for rr in range(n):
                    check_out(k, out[rr], refs[t].outs[rr], f"{path} t={t} {k}/{r} step {s} rank {rr}")
    finally:
        w.destroy()


@pytest.mark.parametrize("fits", [True, False])
def test_onchip_capacity_edge(fits):
    """The largest bucket the on-chip kernel takes (#SMs CTAs of 12 tiles) and
    one tile more (the chain): both bit-exact; the first is one h1 launch."""
    E = esp()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 2
    N = (sms // n) * 12 * 4096 - 1000 + (0 if fits else 4096)
    w = E.World.sim(n, 0)
    try:
        ctx = E.Ctx(w, "dgc", "allgather", N, tensor_id=22, ratio=0.01)
        cfg = O.Cfg("dgc", 0.01)
        st = O.new_states(n, N, "allgather", cfg)
        for s in range(2):
            grads = [gradient(N, step=s, rank=r, tensor=22) for r in range(n)]
            ref = O.sync("allgather", cfg, grads, st, tensor_id=22)
            g = upload(grads)
            l0 = E.esp_launch_count()
            E.esp_sync(w, ctx, g)
            torch.cuda.synchronize()
            if s == 0:   # (later calls replay a CUDA graph, which counts nothing)
                launches = E.esp_launch_count() - l0
            out = g.cpu().numpy().reshape(n, N)
            for r in range(n):
                check_out("dgc", out[r], ref.outs[r], f"fits={fits} step {s} rank {r}")
        _, rg, _ = ctx.get_state()
        for r in range(n):
            assert np.array_equal(bits(rg[r]), bits(st[r].r)), f"residual rank {r}"
        if fits:
            assert launches <= 5, launches
        else:
            assert launches >= 8, launches
    finally:
        w.destroy()


@pytest.mark.parametrize("mode", ["equal", "mixed"])
@pytest.mark.parametrize("ratio", [0.01, 0.3])
def test_onchip_many_members(mode, ratio):
    """Round 1's bin holding more than 16384 keys of a segment (all-equal
    magnitudes; a 30% ratio on a wide segment) takes the distributed rounds 3
    and count with two more barriers; few members, the redundant finish."""
    run_sim("dgc", "allgather", 2, 600_001, steps=2, ratio=ratio, dist="D4", mode=mode)
