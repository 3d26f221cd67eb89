#!/usr/bin/env python
"""A bench.py workload at n ranks on ONE GPU through a loopback group (the n
ranks' fused job tables on one device, launched rank by rank): the per-rank
kernels of an n-rank step (h2 over n pieces, a7, pushes) can then be listed
and profiled with ncu, which must not run multi-rank commands.  Gradients are
device-generated (timing / profiling only, no parity).
usage: loopback_probe.py [--workload W] [--n 4] [--steps 3]"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2205_14465_b200 import esp as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert_large_dgc_allgather")
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    model, rule = bench.workload(args.workload, args.n)
    sizes = bench.shapes.numels(model)
    ws = E.World.loopback(args.n)
    ctxs = []
    for r in range(args.n):
        cs = []
        for t, N in enumerate(sizes):
            k, ra, ro, ex = bench.opt(rule, N)
            cs.append(E.Ctx(ws[r], k, ro, N, tensor_id=t, ratio=ra, **ex))
        ctxs.append(cs)
    grads = [[torch.randn(N, device="cuda") * 1e-2 for N in sizes] for _ in range(args.n)]
    E.esp_sync_many_loopback(ws, ctxs, grads)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        E.esp_sync_many_loopback(ws, ctxs, grads)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(f"{args.workload} loopback n={args.n}: {ms:.3f} ms per step for all ranks "
          f"({ms / args.n:.3f} ms per rank serialised)", flush=True)
    for cs in ctxs:
        for c in cs:
            c.destroy()
    for w in ws:
        w.destroy()


if __name__ == "__main__":
    main()
