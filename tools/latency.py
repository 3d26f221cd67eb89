#!/usr/bin/env python
"""Per-call latency of esp_compress / esp_decompress / esp_sync at small sizes:
host time (wall clock per call, calls back to back) vs device time (the calls
are enqueued behind a long sleep kernel, so the GPU runs them back to back
without waiting for the host).  Shows whether small messages are host- or
device-bound (the paper's "constant overhead to launch GPU kernels").

    python tools/latency.py
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_14465_b200 import esp as E  # noqa: E402


def measure(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    host = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e9 * max(1.0, host * reps / 1e6 * 2)))   # keep the GPU busy while enqueueing
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / reps * 1e3
    return host, dev


def main():
    torch.cuda.set_device(0)
    w = E.World.nccl_single(0)
    sim = E.World.sim(2, 0)
    print(f"{'case':44s} {'host us/call':>12s} {'device us/call':>15s}")
    for kind, ratio in (("dgc", 0.01), ("randomk", 0.01), ("efsignsgd", 1.0)):
        for N in (256, 1 << 20):
            c = E.Ctx(w, kind, "allgather", N, ratio=ratio)
            g = torch.randn(N, device="cuda")
            pay = torch.empty(c.payload_bytes, dtype=torch.uint8, device="cuda")
            out = torch.empty(N, device="cuda")
            h, d = measure(lambda: E.esp_compress(c, g, pay))
            print(f"{kind + ' compress N=' + str(N):44s} {h:12.1f} {d:15.1f}")
            h, d = measure(lambda: E.esp_decompress(c, [pay], out))
            print(f"{kind + ' decompress N=' + str(N):44s} {h:12.1f} {d:15.1f}")
            c.destroy()
    # BASELINE config 1: 1M fp32, DGC 1% + EF, Allgather, n = 2 simulated ranks
    for N in (1 << 20, 10 ** 6):
        c = E.Ctx(sim, "dgc", "allgather", N, ratio=0.01)
        g = torch.randn(2 * N, device="cuda")
        h, d = measure(lambda: E.esp_sync(sim, c, g))
        print(f"{'config 1 sync (sim n=2) N=' + str(N):44s} {h:12.1f} {d:15.1f}")
        c.destroy()
    w.destroy()
    sim.destroy()


if __name__ == "__main__":
    main()
