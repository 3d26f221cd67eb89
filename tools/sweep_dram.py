#!/usr/bin/env python
"""Config-2 DRAM evidence: one esp_compress (h1) and one
8-piece esp_decompress (h2) per compressor at 2^20, 2^26 and 2^30 bytes of fp32
input, after one warm-up of each, for ncu's dram__bytes_{read,write}.sum and
gpu__time_duration.sum on every kernel:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --profile-from-start off --csv --log-file sweep_dram.csv python tools/sweep_dram.py
    python tools/sweep_dram.py --summary sweep_dram.csv
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
    mark = torch.empty(1, device="cuda")
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
            torch.cuda.profiler.start()        # ncu --profile-from-start off: measured calls only
            mark.fill_(float(ex))              # separator kernel (at::...Fill) before each config
            E.esp_compress(c, g, pay)
            E.esp_decompress(c, [pay] * 8, out)
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
            c.destroy()
            del g, out, pay
            torch.cuda.empty_cache()
    w.destroy()


CONFIGS = [(k, ex) for k in ("dgc", "randomk", "efsignsgd") for ex in (20, 26, 30)]


def summary(path):
    """Per config: each kernel's time and DRAM bytes, and the h1 + h2 total
    against the algorithmic bytes (input 4 B/elem: h1 12 B/elem with EF;
    h2: 8 pieces read + 4 B/elem written)."""
    import csv
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    hdr = next(r for r in csv.reader(open(path)) if r and r[0] == "ID")
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    launches = {}
    order = []
    for r in rows:
        key = int(r[0])
        if key not in launches:
            launches[key] = {"name": r[ki]}
            order.append(key)
        v = float(r[vi].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1)
        launches[key][r[mi]] = v * scale
    groups, cur = [], None
    for key in order:
        L = launches[key]
        if "Fill" in L["name"]:
            cur = []
            groups.append(cur)
        elif cur is not None:
            cur.append(L)
    print(f"{'config':<18}{'kernel':<44}{'us':>9}{'DRAM rd MB':>12}{'DRAM wr MB':>12}")
    for (kind, ex), g in zip(CONFIGS, groups):
        tot_t = tot_b = 0.0
        for L in g:
            t = L.get("gpu__time_duration.sum", 0.0)
            rd = L.get("dram__bytes_read.sum", 0.0) / 1e6
            wr = L.get("dram__bytes_write.sum", 0.0) / 1e6
            tot_t += t
            tot_b += rd + wr
            print(f"{kind + ' 2^' + str(ex) + ' B':<18}{L['name'][:43]:<44}{t:>9.1f}{rd:>12.2f}{wr:>12.2f}")
        print(f"{'':<18}{'total':<44}{tot_t:>9.1f}{'':>12}{tot_b:>12.2f}  ({tot_b / max(tot_t, 1e-9):.2f} TB/s DRAM)")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summary":
        summary(sys.argv[2])
    else:
        main()
