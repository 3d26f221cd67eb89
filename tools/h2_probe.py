#!/usr/bin/env python
"""h2 at 2^28 elements (the config-2 sweep's 2^30-byte point) for ncu: EFSignSGD
with 1 and 8 pieces, DGC 1% with 1 and 8 pieces, Randomk 1% with 8 pieces;
`--reps` esp_decompress calls each after one warm-up, device-timed."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_14465_b200 import esp as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=1 << 28)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    w = E.World.nccl_single(0)
    n = args.n
    out = torch.empty(n, device="cuda")
    for kind, ratio in (("efsignsgd", 1.0), ("dgc", 0.01), ("randomk", 0.01)):
        c = E.Ctx(w, kind, "allgather", n, tensor_id=1, ratio=ratio)
        g = torch.randn(n, device="cuda") * 1e-2
        pay = E.esp_compress(c, g)
        for npieces in (1, 8):
            if kind == "randomk" and npieces == 1:
                continue
            pieces = [pay] * npieces
            E.esp_decompress(c, pieces, out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                E.esp_decompress(c, pieces, out)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.reps
            byts = 4 * n + npieces * c.payload_bytes
            print(f"{kind} h2 x{npieces}: {us:.1f} us, {byts / us / 1e3:.0f} GB/s algorithmic", flush=True)
        c.destroy()
        del g, pay
    w.destroy()


if __name__ == "__main__":
    main()
