#!/usr/bin/env python
"""BASELINE config 1 as a stand-alone program (for ncu launch lists): one
2^20-element fp32 gradient, DGC top-1% with error feedback, Allgather, n = 2
simulated ranks; `--reps` back-to-back esp_sync calls after 10 warm-up calls.

    python tools/config1.py [--reps 20]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_14465_b200 import esp as E  # noqa: E402
from synth.values import gradient  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    N, n = 1 << 20, 2
    w = E.World.sim(n, 0)
    c = E.Ctx(w, "dgc", "allgather", N, tensor_id=0, ratio=0.01)
    g = torch.from_numpy(np.concatenate([gradient(N, rank=r) for r in range(n)])).cuda()
    for _ in range(10):
        E.esp_sync(w, c, g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        E.esp_sync(w, c, g)
    e1.record()
    torch.cuda.synchronize()
    print(f"config 1: {e0.elapsed_time(e1) * 1e3 / args.reps:.1f} us per esp_sync (device events, back to back)")
    w.destroy()


if __name__ == "__main__":
    main()
