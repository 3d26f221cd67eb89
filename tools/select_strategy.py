#!/usr/bin/env python
"""NEXT-3 CLI: per-tensor strategy for a model from the measured B200 cost
curves (paper_2205_14465_b200/strategy.py) vs config 5's fixed rule; writes
profiles/r01_strategy_<model>_n<n>.json.

    python tools/select_strategy.py [--model gpt2_medium] [--n 8] [--B 7.7e11]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_14465_b200 import strategy as S  # noqa: E402
from synth import shapes  # noqa: E402


def fixed_option(N):
    k = shapes.gpt2_medium_mixed_rule(N)
    return {"dgc": ("dgc", 0.01, "allgather", 0), "efsignsgd": ("efsignsgd", 1.0, "alltoall_allgather", 2),
            "none": ("none", 1.0, "allreduce", 0)}[k]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt2_medium")
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--B", type=float, default=7.7e11, help="bytes/s per direction (measured NVLink 5)")
    ap.add_argument("--cost-model", dest="cost_model", default="paper", choices=["paper", "bucketed"])
    ap.add_argument("--algorithm", default="dgc", help="the GC algorithm (P:1217); 'all' = every algorithm")
    args = ap.parse_args()
    alg = None if args.algorithm == "all" else args.algorithm
    sel = S.Selector(args.n, args.B, model=args.cost_model, algorithm=alg)
    full = S.Selector(args.n, args.B, model=args.cost_model, algorithm=None)   # prices the fixed rule
    sizes = shapes.numels(args.model)
    per_size, total, total_fixed = {}, 0.0, 0.0
    for N in sorted(set(sizes), reverse=True):   # Property #2: larger tensors first
        best, t = sel.choose(N)
        fo = fixed_option(N) if args.model == "gpt2_medium" else ("none", 1.0, "allreduce", 0)
        fi = [c[:4] for c in full.candidates].index(fo)
        tf = full.predicted(fi, N)
        cnt = sizes.count(N)
        per_size[str(N)] = {"count": cnt, "selected": sel.candidates[best][:4], "predicted_s": t,
                            "fixed_rule": fo, "fixed_rule_predicted_s": tf}
        total += cnt * t
        total_fixed += cnt * tf
    out = {"model": args.model, "n": args.n, "B": args.B, "sweep": "profiles/r01_sweep.json",
           "objective": "sum of per-tensor sync times (cost table P:38-43 + fitted h1/h2, reading R21)",
           "predicted_total_s": total, "fixed_rule_predicted_total_s": total_fixed, "per_size": per_size}
    suffix = ("" if args.cost_model == "paper" else "_bucketed") + ("" if args.algorithm == "dgc" else "_" + args.algorithm)
    out["cost_model"] = args.cost_model
    out["algorithm"] = args.algorithm
    path = os.path.join(ROOT, "profiles", f"r01_strategy_{args.model}_n{args.n}{suffix}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    for N, v in per_size.items():
        print(f"N={N:>10} x{v['count']:<4} selected {'/'.join(map(str, v['selected'])):36s} "
              f"{v['predicted_s'] * 1e6:9.1f} us   fixed {'/'.join(map(str, v['fixed_rule'])):36s} "
              f"{v['fixed_rule_predicted_s'] * 1e6:9.1f} us")
    print(f"predicted total: selected {total * 1e3:.3f} ms, fixed rule {total_fixed * 1e3:.3f} ms -> {path}")


if __name__ == "__main__":
    main()
