#!/usr/bin/env python
"""h1 (esp_compress) of one tensor, device-timed, for launch lists / ncu:
`h1_probe.py --kind dgc --ratio 0.01 --n 268435456 --reps 3`."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_14465_b200 import esp as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="dgc")
    ap.add_argument("--ratio", type=float, default=0.01)
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    w = E.World.nccl_single(0)
    c = E.Ctx(w, args.kind, "allgather", args.n, tensor_id=1, ratio=args.ratio)
    g = torch.randn(args.n, device="cuda") * 1e-2
    pay = torch.empty(c.payload_bytes, dtype=torch.uint8, device="cuda")
    E.esp_compress(c, g, pay)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        E.esp_compress(c, g, pay)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.reps
    print(f"{args.kind} {args.ratio} h1 n={args.n}: {us:.1f} us, {12 * args.n / us / 1e3:.0f} GB/s (12 B/elem)", flush=True)
    c.destroy()
    w.destroy()


if __name__ == "__main__":
    main()
