#!/usr/bin/env python
"""Markdown table of bench.py JSON lines: `bench_table.py file.json ...`
(the last line of each file; files without a line are listed as failed)."""
import json
import sys


def fmt(x, nd=3):
    return f"{x:.{nd}f}" if isinstance(x, (int, float)) else ("—" if x is None else str(x))


def main():
    print("| file | workload | n | GB/s per rank | GB/s aggregate | ms/step | e2e GB/s | h1 frac | comm ms (serialised) | link GB/s | link frac |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for f in sys.argv[1:]:
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except (OSError, IndexError, ValueError):
            print(f"| {f} | failed | | | | | | | | | |")
            continue
        link = d.get("link") or {}
        ph = d.get("phases_ms_serialised") or {}
        print(f"| {f.split('/')[-1]} | {d['config'].get('workload')} | {d['n_gpus']} | {fmt(d.get('value_per_rank'), 1)} "
              f"| {fmt(d['value'], 1)} | {fmt(d['ms_per_step'], 4)} | {fmt((d.get('e2e') or {}).get('value'), 1)} "
              f"| {fmt(d['roofline']['frac'])} | {fmt(ph.get('comm_ms'))} | {fmt(link.get('achieved_GBps'), 1)} "
              f"| {fmt(link.get('frac'))} |")


if __name__ == "__main__":
    main()
