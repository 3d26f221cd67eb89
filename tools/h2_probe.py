#!/usr/bin/env python
"""h2 at 2^28 elements (the config-2 sweep's 2^30-byte point) for ncu:
EFSignSGD, DGC 1% and Randomk 1% with 1 and 8 pieces (default), or the
compressor / ratio / piece counts given; `--reps` esp_decompress calls each
after one warm-up, device-timed.  With --distinct every piece is the payload of
a different gradient (as at n ranks), else one payload is repeated."""
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
    ap.add_argument("--only", default="", help="kind:ratio, e.g. dgc:0.001 (default: the three compressors)")
    ap.add_argument("--pieces", default="1,8")
    ap.add_argument("--distinct", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    w = E.World.nccl_single(0)
    n = args.n
    out = torch.empty(n, device="cuda")
    runs = [("efsignsgd", 1.0), ("dgc", 0.01), ("randomk", 0.01)]
    if args.only:
        k, r = args.only.split(":")
        runs = [(k, float(r))]
    counts = [int(x) for x in args.pieces.split(",")]
    for kind, ratio in runs:
        c = E.Ctx(w, kind, "allgather", n, tensor_id=1, ratio=ratio)
        npay = max(counts) if args.distinct else 1
        pays = []
        for i in range(npay):
            g = torch.randn(n, device="cuda") * 1e-2
            pays.append(E.esp_compress(c, g))
            del g
        for npieces in counts:
            if kind == "randomk" and npieces == 1 and not args.only:
                continue
            pieces = [pays[i % npay] for i in range(npieces)]
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
            print(f"{kind} {ratio} h2 x{npieces}{' distinct' if args.distinct else ''}: {us:.1f} us, "
                  f"{byts / us / 1e3:.0f} GB/s algorithmic", flush=True)
        c.destroy()
        del pays
    w.destroy()


if __name__ == "__main__":
    main()
