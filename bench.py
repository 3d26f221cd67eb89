#!/usr/bin/env python
"""Benchmark of the compressed gradient-synchronisation hot path on B200.

Metric (BASELINE.json): compressed gradient-sync GB/s (device-timed, max over
ranks).  Per rank, one step synchronises that rank's whole gradient set,
sum over tensors of 4 * numel bytes, with one esp_sync_many (h1 -> collective
-> h2); t_step = max over ranks of its CUDA-event time, inputs resident in HBM.
`value` is the whole job's throughput, the gradient bytes all n ranks
synchronised per step / t_step (weak scaling: each rank syncs its own full
gradient set); `value_per_rank` = 4 * sum numel / t_step is BASELINE.md's
per-rank figure (value / n).

    python bench.py [--gpus N --steps K --warmup W --workload NAME]
        (--gpus N > 1 without a torchrun environment re-launches itself under
         torch.distributed.run with N ranks, one per GPU, NCCL)
    python bench.py --impl reference ...                  (the CPU oracle, host cores)

Default workload = BASELINE config 4: BERT-large (BertForPreTraining shapes,
398 tensors, 336,226,108 params per rank), DGC top-0.1% with error feedback,
Allgather.  Synthetic gradients (synth/values.py, D1), generated per rank.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
from synth import shapes  # noqa: E402
from synth.values import BASE_SEED, gradient  # noqa: E402

WORKLOADS = {
    # name: (model, per-tensor rule numel -> (kind, ratio, routine[, extra ctx options]))
    "bert_large_dgc_allgather": ("bert_large", lambda N: ("dgc", 0.001, "allgather")),
    "bert_large_dgc_alltoall": ("bert_large", lambda N: ("dgc", 0.001, "alltoall_allgather")),
    "resnet50_efsignsgd_alltoall": ("resnet50", lambda N: ("efsignsgd", 1.0, "alltoall_allgather")),
    "gpt2_medium_mixed": ("gpt2_medium", lambda N: {
        "dgc": ("dgc", 0.01, "allgather"),
        "efsignsgd": ("efsignsgd", 1.0, "alltoall_allgather"),
        "none": ("none", 1.0, "allreduce")}[shapes.gpt2_medium_mixed_rule(N)]),
    # DGC with momentum correction (R20, NEXT-2): 20 B/elem streaming pass
    "bert_large_dgc_momentum_allgather": ("bert_large", lambda N: ("dgc", 0.001, "allgather", {"momentum": 0.9})),
    # NEXT-3: per-size options chosen by the cost model over the measured curves
    # (paper_2205_14465_b200/strategy.py) for the run's rank count
    "gpt2_medium_selected": ("gpt2_medium", ("selected", "paper", "dgc")),
    "gpt2_medium_selected_bucketed": ("gpt2_medium", ("selected", "bucketed", "dgc")),
    "gpt2_medium_selected_bucketed_all": ("gpt2_medium", ("selected", "bucketed", None)),
    # NEXT-4: hierarchical communication, "machines" of 2 GPUs (1 when n is
    # odd): intra Reduce-scatter, inter-machine DGC 0.1% Allgather per shard,
    # intra Allgather (esp_world_create_hier)
    "bert_large_dgc_hier2": ("bert_large", lambda N: ("dgc", 0.001, "allgather")),
}
HIER_GROUP = {"bert_large_dgc_hier2": 2}


def hier_group(name, n):
    g = HIER_GROUP.get(name, 0)
    return (g if n % g == 0 else 1) if g else 0


def workload(name, n):
    """-> (model, rule) with the selected strategy resolved for n ranks."""
    model, rule = WORKLOADS[name]
    if isinstance(rule, tuple) and rule[0] == "selected":
        from paper_2205_14465_b200 import strategy
        rule = strategy.Selector(max(1, n), model=rule[1], algorithm=rule[2]).rule
    return model, rule


def opt(rule, N):
    """-> (kind, ratio, routine, extra) of a workload rule."""
    r = rule(N)
    return (*r, {}) if len(r) == 3 else r


def strategy_str(rule, N):
    k, ra, ro, ex = opt(rule, N)
    return "/".join([k, str(ra), ro] + [f"{a}={b}" for a, b in sorted(ex.items())])
DEFAULT = "bert_large_dgc_allgather"
E2E_CHUNKS = 4   # tensor groups of the pipelined e2e loop


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ NVLink counters
def nvlink_bytes(gpu_index: int):
    """(tx, rx) bytes over all NVLinks of the GPU so far, from NVML's NVLink
    throughput counters (data payload, KiB) or, where those are missing, the
    per-link byte counters; None if NVML offers neither."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(gpu_index)
        vals = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                               nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
        if all(v.nvmlReturn == 0 for v in vals):
            return {"tx": int(vals[0].value.ullVal) * 1024, "rx": int(vals[1].value.ullVal) * 1024,
                    "source": "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (KiB)"}
        tx = rx = 0
        for link in range(18):
            v = nv.nvmlDeviceGetFieldValues(h, [(nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, link),
                                                (nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, link)])
            if v[0].nvmlReturn == 0:
                tx += int(v[0].value.ullVal)
            if v[1].nvmlReturn == 0:
                rx += int(v[1].value.ullVal)
        return {"tx": tx, "rx": rx, "source": "NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES per link"}
    except Exception as e:   # noqa: BLE001 (diagnostic only)
        return {"error": f"{type(e).__name__}: {e}"}


# ------------------------------------------------------------------ config-1 latency
def latency_config1(E, device: int, reps: int = 200):
    """BASELINE config 1 as a latency probe: one 2^20-element fp32 gradient, DGC
    top-1% with error feedback, Allgather, n = 2 simulated ranks on this GPU
    (sim world: both ranks' h1 / h2 kernels, the collective is two D2D copies).
    Mean device time per esp_sync over `reps` back-to-back calls (inputs L2-
    resident: this probes the per-call launch chain)."""
    import torch
    N, n = 1 << 20, 2
    w = E.World.sim(n, device)
    c = E.Ctx(w, "dgc", "allgather", N, tensor_id=0, ratio=0.01)
    g = torch.from_numpy(__import__("numpy").concatenate([gradient(N, rank=r) for r in range(n)])).cuda()
    for _ in range(10):
        E.esp_sync(w, c, g)
    l0 = E.esp_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        E.esp_sync(w, c, g)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    launches = (E.esp_launch_count() - l0) / reps
    w.destroy()
    hbm = 2 * (12 * N + 4 * N)   # per rank: h1 12 B/elem + h2 4 B/elem
    return {"workload": "config 1: 2^20 fp32, DGC 1%, EF, Allgather, sim n=2", "us_per_sync": us,
            "gbs": n * 4 * N / (us * 1e-6) / 1e9, "kernel_launches_per_sync": launches,
            "roofline_us": hbm / (peaks()[0]["hbm_gbs"] * 1e3), "reps": reps}


# ------------------------------------------------------------------ output
_JSON_FD = None


def _claim_stdout():
    """The JSON line must be the only stdout output: keep a private handle on
    the real stdout and point fd 1 (C libraries such as NCCL print there) at
    stderr."""
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def emit(line: dict):
    fd = _JSON_FD if _JSON_FD is not None else 1
    os.write(fd, (json.dumps(line) + "\n").encode())


# ------------------------------------------------------------------ dist helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def max_over_ranks_vec(xs, ws):
    if ws == 1:
        return list(xs)
    import torch
    import torch.distributed as dist
    t = torch.tensor(xs, dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The oracle (oracle/esp_oracle.py) as it stands, on the host cores: each
    step syncs a bounded sample of the workload's tensors (n ranks simulated)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import esp_oracle as O
    model, rule = workload(args.workload, ws)
    names = [nm for nm, _ in shapes.MODELS[model]()]
    sizes = shapes.numels(model)
    # sample: the first ~4M elements of encoder/transformer weights after the embeddings
    idx, tot = [], 0
    for i, (nm, N) in enumerate(zip(names, sizes)):
        if i == 0 or "embed" in nm or "wte" in nm or "wpe" in nm:
            continue
        idx.append(i)
        tot += N
        if tot >= 4_000_000:
            break
    n = max(1, args.gpus)
    cores = os.cpu_count() or 1
    jobs = [(args.workload, n, i, sizes[i]) for i in idx]
    # one worker process per host core, each owning a share of the tensors (the
    # oracle is single-threaded numpy); every step syncs every sampled tensor once
    with multiprocessing.get_context("fork").Pool(min(cores, len(jobs)), initializer=_oracle_worker_init) as pool:
        pool.map(_oracle_job, jobs)                      # builds each worker's states
        for _ in range(args.warmup):
            pool.map(_oracle_job, jobs)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_oracle_job, jobs)
        dt = (time.perf_counter() - t0) / args.steps
    value = n * 4 * tot / dt / 1e9
    sample = (f"{len(idx)} tensors of {args.workload} ({tot} elements per rank, first non-embedding tensors), "
              f"n={n} ranks simulated, {min(cores, len(jobs))} worker processes on {cores} host cores ({_cpu_model()})")
    line = {
        "impl": "reference", "metric": "compressed gradient-sync GB/s", "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": args.workload, "parallelism": f"dp{n}"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": min(cores, len(jobs)), "kind": "oracle",
                         "sample": sample, "host": {"nproc": cores, "cpu_model": _cpu_model()}},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


# oracle worker processes (fork): each keeps the EF states of the tensors it was
# handed, so repeated steps carry error feedback like the real path
_W = {}


def _oracle_worker_init():
    os.environ["OMP_NUM_THREADS"] = "1"


def _oracle_job(job):
    from oracle import esp_oracle as O
    name, n, i, N = job
    if ("rule", name, n) not in _W:
        _W[("rule", name, n)] = workload(name, n)[1]
    rule = _W[("rule", name, n)]
    kind, ratio, routine, ex = opt(rule, N)
    cfg = O.Cfg(kind, ratio, **ex)
    g = hier_group(name, n)
    if (name, i) not in _W:
        st = O.new_states_hier(n, N, routine, cfg, g) if g else O.new_states(n, N, routine, cfg)
        _W[(name, i)] = ([gradient(N, rank=r, tensor=i) for r in range(n)], st)
    grads, st = _W[(name, i)]
    t0 = time.perf_counter()
    if g:
        O.sync_hierarchical(routine, cfg, grads, st, g, tensor_id=i)
    else:
        O.sync(routine, cfg, grads, st, tensor_id=i)
    return time.perf_counter() - t0


def cpu_baseline(args, model, rule, sizes, names, n):
    """The oracle timed on this host on a bounded sample (~10-30 s of CPU work):
    single-threaded, then one worker process per host core over the same
    tensors (the oracle itself is single-threaded numpy)."""
    idx, tot = [], 0
    for i, nm in enumerate(names):
        if any(s in nm for s in ("layer.0.", "layer.1.", "layer.2.", "layer1.", "h.0.", "h.1.")):
            idx.append(i)
            tot += sizes[i]
    if not idx:
        idx = list(range(min(20, len(sizes))))
        tot = sum(sizes[i] for i in idx)
    jobs = [(args.workload, n, i, sizes[i]) for i in idx]
    t1 = sum(_oracle_job(j) for j in jobs)          # one core (states built on the first call, untimed)
    t1 = sum(_oracle_job(j) for j in jobs)
    cores = os.cpu_count() or 1
    nw = min(cores, len(jobs))
    with multiprocessing.get_context("fork").Pool(nw, initializer=_oracle_worker_init) as pool:
        pool.map(_oracle_job, jobs)
        t0 = time.perf_counter()
        pool.map(_oracle_job, jobs)
        tall = time.perf_counter() - t0
    return {"value": n * 4 * tot / tall / 1e9, "unit": "GB/s", "cores": nw, "kind": "oracle",
            "single_thread_value": n * 4 * tot / t1 / 1e9,
            "host": {"nproc": cores, "cpu_model": _cpu_model()},
            "sample": f"{len(idx)} tensors ({tot} elements per rank) of the first layers, n={n} ranks simulated; "
                      f"value: {nw} worker processes over the tensors ({tall:.1f} s); single thread {t1:.1f} s"}


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="espresso", choices=["espresso", "reference"])
    ap.add_argument("--workload", default=DEFAULT, choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--bucket-elems", type=int, default=0)
    ap.add_argument("--phases", action="store_true", help="print a serialised h1/comm/mid/h2 breakdown to stderr")
    ap.add_argument("--no-latency", action="store_true", help="skip the config-1 latency probe")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        # one process per GPU: re-launch under torch.distributed.run; rank 0 prints the line
        import socket
        for attempt in range(3):   # a fresh port again if the rendezvous never came up (port taken meanwhile)
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
            p = subprocess.run(cmd, stdout=subprocess.PIPE, text=True)
            sys.stdout.write(p.stdout)
            sys.stdout.flush()
            if p.returncode == 0 or p.stdout.strip():
                break
        sys.exit(p.returncode)
    _claim_stdout()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2205_14465_b200 import esp as E

    model, rule = workload(args.workload, ws)
    names = [nm for nm, _ in shapes.MODELS[model]()]
    sizes = shapes.numels(model)
    total = sum(sizes)
    world = E.World.nccl(local) if ws > 1 else E.World.nccl_single(local)
    flat_world = None
    if hier_group(args.workload, ws):
        flat_world, world = world, world.hier(hier_group(args.workload, ws))
    if args.bucket_elems:
        world.set_bucket_elems(args.bucket_elems)
    ctxs = []
    for t, N in enumerate(sizes):
        kind, ratio, routine, ex = opt(rule, N)
        ctxs.append(E.Ctx(world, kind, routine, N, tensor_id=t, ratio=ratio, **ex))

    # gradients: one flat buffer, tensors at 16-byte aligned offsets
    offs, o = [], 0
    for N in sizes:
        offs.append(o)
        o += (N + 3) // 4 * 4
    host = torch.empty(o, dtype=torch.float32).pin_memory()
    hv = host.numpy()
    for t, N in enumerate(sizes):
        hv[offs[t]:offs[t] + N] = gradient(N, seed=BASE_SEED, rank=rank, tensor=t)
    g0 = host.cuda()
    g = torch.empty_like(g0)
    views = [g[offs[t]:offs[t] + N] for t, N in enumerate(sizes)]
    stream = torch.cuda.current_stream()

    def step():
        E.esp_sync_many(world, ctxs, views, stream)

    # L2 hygiene: before every timed step, after restoring the gradients, write
    # a buffer of twice the 126 MB L2 so that no input of the step starts in L2
    # (the restore itself leaves the last ~126 MB of g resident otherwise)
    flush = torch.empty(2 * 126 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")

    def restore():
        g.copy_(g0)
        flush.fill_(1.0)

    for _ in range(args.warmup):
        restore()
        step()
    torch.cuda.synchronize()
    barrier(ws)

    # ---- timed region: K steps, per-step CUDA events on the launching stream.
    # Before every step: the input restore (the "backward pass" that produces
    # fresh gradients), the L2 flush and, with several ranks, a barrier ON THE
    # GPU (a one-element NCCL all-reduce on the stream), so that every rank's
    # step starts together while the host keeps enqueueing ahead; the step's
    # time is the max over ranks of its event time
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    world.set_probe(True)
    launches0 = E.esp_launch_count()
    barrier(ws)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    nvl0 = nvlink_bytes(local) if ws > 1 else None
    gbar = torch.zeros(1, device="cuda")
    for i in range(args.steps):
        restore()
        if ws > 1:
            import torch.distributed as dist
            dist.all_reduce(gbar)   # device-side barrier: the step starts when every rank got here
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    wall = time.perf_counter() - w0
    nvl1 = nvlink_bytes(local) if ws > 1 else None
    launches = E.esp_launch_count() - launches0
    probe_ms, probe_n, probe_bytes = world.probe_read()
    world.set_probe(False)
    clk = clocks.stop() if clocks else None
    step_ms = max_over_ranks_vec([a.elapsed_time(b) for a, b in ev], ws)   # per step, max over ranks
    t_mean = sum(step_ms) / len(step_ms)
    t_med = statistics.median(step_ms)

    # ---- optional per-phase breakdown (serialised phases; diagnostics on stderr)
    phases = None
    counters = None
    if args.phases or ws > 1:
        world.set_timing(True)
        world.reset_counters()
        acc = {}
        for _ in range(5):
            restore()
            step()
            for k_, v_ in world.last_timing().items():
                acc[k_] = acc.get(k_, 0.0) + v_ / 5
        world.set_timing(False)
        phases = {k_: max_over_ranks(v_, ws) for k_, v_ in acc.items()}
        counters = world.counters()
        if rank == 0 and args.phases:
            print("phases (ms, serialised, max over ranks):", json.dumps(phases), file=sys.stderr)

    # ---- e2e: host gradients (pinned) -> device, sync, result -> host, through
    # the public API.  The tensor set is synchronised in E2E_CHUNKS groups of
    # tensors (esp_sync_many per group; per-tensor results do not depend on the
    # grouping) so that the H2D copy of group c + 1, the sync of group c and the
    # D2H copy of group c - 1 overlap (PCIe is full duplex); every step still
    # copies all of its inputs in and all of its results out.
    out_host = torch.empty_like(host).pin_memory() if args.e2e_steps else None
    e2e_ms = None
    if args.e2e_steps:
        C_ = E2E_CHUNKS
        bounds, acc_b, tgt = [0], 0, 4 * o / C_
        for t, N in enumerate(sizes):
            acc_b += 4 * N
            if acc_b >= tgt * len(bounds) and len(bounds) < C_ and t + 1 < len(sizes):
                bounds.append(t + 1)
        bounds.append(len(sizes))
        groups = [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)]
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in groups]
        ev_done = [torch.cuda.Event() for _ in groups]
        ev_out = [torch.cuda.Event() for _ in groups]

        def span(a, b_):
            lo = offs[a]
            hi = offs[b_ - 1] + sizes[b_ - 1]
            return lo, hi

        def e2e_step(first):
            for c, (a, b_) in enumerate(groups):
                lo, hi = span(a, b_)
                with torch.cuda.stream(h2d_s):
                    if not first:
                        h2d_s.wait_event(ev_out[c])   # the previous step's result left this range
                    g[lo:hi].copy_(host[lo:hi], non_blocking=True)
                    ev_in[c].record(h2d_s)
                stream.wait_event(ev_in[c])
                E.esp_sync_many(world, ctxs[a:b_], views[a:b_], stream)
                ev_done[c].record(stream)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(ev_done[c])
                    out_host[lo:hi].copy_(g[lo:hi], non_blocking=True)
                    ev_out[c].record(d2h_s)

        e2e_step(True)   # builds the per-group plans (untimed)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(ws)
        e0.record(stream)
        h2d_s.wait_event(e0)
        for i in range(args.e2e_steps):
            e2e_step(False)
        for c in range(len(groups)):
            stream.wait_event(ev_out[c])
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps, ws)

    if rank == 0:
        pk, pk_src = peaks()
        achieved = probe_bytes / (probe_ms / 1e3) / 1e9 if probe_ms > 0 else None
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_stream_traffic.json")) as f:
                tr = json.load(f)
            if tr.get("workload") == args.workload:
                traffic = tr.get("dram_bytes_per_launch")
        except OSError:
            pass
        bytes_per_rank = 4 * total
        value = ws * bytes_per_rank / (t_mean / 1e3) / 1e9
        link = None
        if ws > 1:
            # NVLink: bytes this rank pushed per step (fused collectives) and the
            # cost-table volume, against the serialised comm phase and the link
            push_b = counters["pushed"] / 5
            logical = counters["sent"] / 5
            comm_ms = phases.get("comm_ms") if phases else None
            link = {"bytes_pushed_per_rank_per_step": push_b, "cost_table_bytes_per_rank_per_step": logical,
                    "comm_ms_serialised": comm_ms,
                    "achieved_GBps": push_b / (comm_ms * 1e-3) / 1e9 if comm_ms else None,
                    "peak_GBps": 770.0, "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
                    "frac": (push_b / (comm_ms * 1e-3) / 1e9) / 770.0 if comm_ms else None}
            if (nvl0 and nvl1 and "tx" in nvl0 and "tx" in nvl1 and nvl1["tx"] == nvl0["tx"]
                    and nvl1["rx"] == nvl0["rx"] and push_b > 0):
                link["nvml"] = ("NVML NVLink byte counters do not advance on this pool; the link bytes are "
                                "measured with ncu nvltx__bytes (profiles/r02_push_nvlink.md)")
            elif nvl0 and nvl1 and "tx" in nvl0 and "tx" in nvl1:
                link["nvml_tx_bytes_per_step"] = (nvl1["tx"] - nvl0["tx"]) / args.steps
                link["nvml_rx_bytes_per_step"] = (nvl1["rx"] - nvl0["rx"]) / args.steps
                link["nvml_source"] = nvl1["source"]
            else:
                link["nvml"] = nvl1
        line = {
            "metric": "compressed gradient-sync GB/s", "value": value, "unit": "GB/s",
            "value_per_rank": bytes_per_rank / (t_mean / 1e3) / 1e9,
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_mean,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": args.workload, "model_shapes": model, "tensors": len(sizes),
                       "params_per_rank": total, "parallelism": f"dp{ws}",
                       "strategy": sorted({strategy_str(rule, N) for N in sizes}),
                       "median_ms_per_step": t_med, "wall_ms_per_step_incl_input_restore": wall * 1e3 / args.steps,
                       "l2": "flushed: after the (untimed) gradient restore, a 252 MB buffer (2x L2) is "
                             "written before every timed step"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"] if achieved else None, "traffic": traffic,
                         "kernel": "h1 streaming pass (dgc_stream_kernel / tma_stream_kernel<SignOp|RandomkOp> / pack_kernel)",
                         "algorithmic_bytes_per_step": probe_bytes / max(1, args.steps),
                         "launches_per_step": probe_n / max(1, args.steps),
                         "kernel_ms_per_step": probe_ms / max(1, args.steps),
                         "kernel_share_of_step": (probe_ms / args.steps) / t_mean,
                         "peak_source": f"{pk_src} MEASURED_PEAKS.json hbm_gbs"},
            "e2e": {"value": ws * bytes_per_rank / (e2e_ms / 1e3) / 1e9 if e2e_ms else None, "unit": "GB/s",
                    "h2d_bytes_per_step": 4 * o, "d2h_bytes_per_step": 4 * o,
                    "ms_per_step": e2e_ms, "pipeline": f"{E2E_CHUNKS} tensor groups, H2D / sync / D2H overlapped"},
            "gpu_launches": launches,
            "clocks": clk,
            **({"phases_ms_serialised": phases} if phases and phases.get("total_ms") else {}),
            # a9: the same step with its phases serialised (events
            # around each) minus the pipelined step = the time the overlap of
            # h1(b+1) / finalize chains with the collective of bucket b hides
            **({"pipelining": {"serialised_ms": phases["total_ms"], "pipelined_ms": t_mean,
                               "hidden_ms": phases["total_ms"] - t_mean}} if phases and phases.get("total_ms") else {}),
            **({"link": link} if link else {}),
        }
        if not args.no_latency:
            line["latency_config1"] = latency_config1(E, local)
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args, model, rule, sizes, names, 1)
        emit(line)
    world.destroy()
    if flat_world is not None:
        flat_world.destroy()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
