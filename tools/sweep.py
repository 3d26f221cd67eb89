#!/usr/bin/env python
"""BASELINE config 2: h1 / h2 cost curves on 1 B200.

For every compressor the paper evaluates and every message size 2^10 .. 2^30
BYTES of fp32 input (reading R16; "2^10, 2^11, ..., 2^30", profiled 100
times and averaged), time esp_compress (h1, EF on) and
esp_decompress with 1 and 8 pieces (h2) through the C ABI with CUDA events:
10 warm-up + 100 timed calls, rotating over enough buffer replicas (>= 2 x L2)
that small sizes are not served from L2.  Output: one JSON document with
CostCurve-shaped samples (size_bytes, mean ns) per (compressor, op)
and the achieved algorithmic GB/s.

    python tools/sweep.py [--min-exp 10 --max-exp 30 --reps 100] > profiles/r01_sweep.json
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2205_14465_b200 import esp as E  # noqa: E402

COMPRESSORS = [("dgc", 0.01), ("dgc", 0.001), ("topk", 0.001), ("randomk", 0.01), ("efsignsgd", 1.0), ("onebit", 1.0)]
L2_BYTES = 126 << 20


def h1_bytes(kind, n):
    """algorithmic HBM bytes of one h1"""
    return 12 * n + (n // 8 if kind in ("efsignsgd", "onebit") else 0)


def timed(fn, reps, warmup, nbuf=1):
    # every buffer replica is touched before timing (its plan is built on first use)
    for i in range(max(warmup, nbuf)):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e6   # ns


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-exp", type=int, default=10)
    ap.add_argument("--max-exp", type=int, default=30)
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    out = {"device": torch.cuda.get_device_name(0), "reps": args.reps, "warmup": args.warmup,
           "sizes": "bytes of fp32 input (R16)", "curves": []}
    w = E.World.nccl_single(0)
    for kind, ratio in COMPRESSORS:
        h1, h2_1, h2_8 = [], [], []
        for ex in range(args.min_exp, args.max_exp + 1):
            nbytes = 1 << ex
            n = nbytes // 4
            reps_buf = max(1, min(32, (2 * L2_BYTES) // nbytes))
            ctxs = [E.Ctx(w, kind, "allgather", n, tensor_id=i, ratio=ratio) for i in range(reps_buf)]
            grads = [torch.randn(n, device="cuda") * 1e-2 for _ in range(reps_buf)]
            pays = [torch.empty(ctxs[0].payload_bytes, dtype=torch.uint8, device="cuda") for _ in range(reps_buf)]
            outs = [torch.empty(n, device="cuda") for _ in range(reps_buf)]
            t1 = timed(lambda i: E.esp_compress(ctxs[i % reps_buf], grads[i % reps_buf], pays[i % reps_buf]),
                       args.reps, args.warmup, reps_buf)
            t21 = timed(lambda i: E.esp_decompress(ctxs[i % reps_buf], [pays[i % reps_buf]], outs[i % reps_buf]),
                        args.reps, args.warmup, reps_buf)
            p8 = [pays[(j) % reps_buf] for j in range(8)]
            t28 = timed(lambda i: E.esp_decompress(ctxs[i % reps_buf], p8, outs[i % reps_buf]), args.reps,
                        args.warmup, reps_buf)
            h1.append({"size_bytes": nbytes, "ns": t1, "gbs": h1_bytes(kind, n) / t1})
            h2_1.append({"size_bytes": nbytes, "ns": t21, "gbs": (4 * n + ctxs[0].payload_bytes) / t21})
            h2_8.append({"size_bytes": nbytes, "ns": t28, "gbs": (4 * n + 8 * ctxs[0].payload_bytes) / t28})
            print(f"{kind} {ratio} 2^{ex}: h1 {t1 / 1e3:.1f} us ({h1[-1]['gbs']:.0f} GB/s), "
                  f"h2x1 {t21 / 1e3:.1f} us, h2x8 {t28 / 1e3:.1f} us", file=sys.stderr, flush=True)
            for c in ctxs:
                c.destroy()
            del grads, pays, outs
            torch.cuda.empty_cache()
        name = f"{kind}_{ratio}"
        out["curves"] += [{"compressor": name, "op": "h1", "device": "gpu", "samples": h1},
                          {"compressor": name, "op": "h2_npieces1", "device": "gpu", "samples": h2_1},
                          {"compressor": name, "op": "h2_npieces8", "device": "gpu", "samples": h2_8}]
    w.destroy()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
