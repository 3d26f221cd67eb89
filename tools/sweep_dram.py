#!/usr/bin/env python
"""Config-2 DRAM evidence: one esp_compress (h1) and one
8-piece esp_decompress (h2) per compressor at 2^20, 2^26 and 2^30 bytes of fp32
input, after one warm-up of each, for ncu's dram__bytes_{read,write}.sum and
gpu__time_duration.sum on every kernel:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --csv --log-file sweep_dram.csv python tools/sweep_dram.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_14465_b200 import esp as E  # noqa: E402


def main():
    torch.cuda.set_device(0)
    w = E.World.nccl_single(0)
    for kind, ratio in (("dgc", 0.01), ("randomk", 0.01), ("efsignsgd", 1.0)):
        for ex in (20, 26, 30):
            n = (1 << ex) // 4
            c = E.Ctx(w, kind, "allgather", n, tensor_id=ex, ratio=ratio)
            g = torch.randn(n, device="cuda") * 1e-2
            out = torch.empty(n, device="cuda")
            pay = E.esp_compress(c, g)                        # warm-up (plan, graph)
            E.esp_decompress(c, [pay] * 8, out)
            torch.cuda.synchronize()
            print(f"MARK {kind} 2^{ex}", flush=True)
            E.esp_compress(c, g, pay)
            E.esp_decompress(c, [pay] * 8, out)
            torch.cuda.synchronize()
            c.destroy()
            del g, out, pay
            torch.cuda.empty_cache()
    w.destroy()


if __name__ == "__main__":
    main()
