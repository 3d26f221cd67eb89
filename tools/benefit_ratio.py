#!/usr/bin/env python
"""Fig. 4 of the paper recomputed on B200: "the ratio of the
reduced communication time to the incurred compression time" per tensor size,
from the measured config-2 curves (profiles/r01_sweep.json) and the cost table
(P:38-43), for n ranks over NVLink 5 at B bytes/s.

    reduced  = T_comm(no compression, Allreduce, 4N) - T_comm(option, M)
    incurred = the option's compression column (h1, h2 from the curves)
    ratio    = reduced / incurred      (> 1: GPU compression pays off)

    python tools/benefit_ratio.py [--n 8] [--B 7.7e11] > profiles/r01_benefit_ratio.txt
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2205_14465_b200 import esp as E  # noqa: E402
from paper_2205_14465_b200 import strategy as S  # noqa: E402

OPTIONS = [("dgc", 0.01, "allgather", 0, "dgc_0.01"), ("dgc", 0.001, "allgather", 0, "dgc_0.001"),
           ("randomk", 0.01, "allreduce", 0, "randomk_0.01"), ("efsignsgd", 1.0, "alltoall_allgather", 2, "efsignsgd_1.0"),
           ("onebit", 1.0, "alltoall_allgather", 2, "onebit_1.0")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--B", type=float, default=7.7e11)
    args = ap.parse_args()
    cv = S.load_curves()
    none = E.make_option("none", 1.0, "allreduce")
    zero = [(1.0, 1e-12)]
    print(f"# benefit ratio of GPU compression on B200, n = {args.n}, B = {args.B:.3g} B/s (Fig. 4, P:1281)")
    print(f"{'bytes':>12s} " + " ".join(f"{o[0] + '_' + str(o[1]) + '/' + o[2][:9]:>26s}" for o in OPTIONS))
    for ex in range(10, 31, 2):
        b = 2 ** ex
        N = b // 4
        t_none = E.option_time(none, N, args.n, args.B)
        row = []
        for kind, ratio, routine, proc, name in OPTIONS:
            o = E.make_option(kind, ratio, routine, h1=cv[(name, "h1")], h2=cv[(name, "h2_npieces1")], process=proc)
            total = E.option_time(o, N, args.n, args.B)
            comm = E.option_time(E.make_option(kind, ratio, routine, h1=zero, h2=zero, process=proc), N, args.n,
                                 args.B)
            row.append((t_none - comm) / max(total - comm, 1e-12))
        print(f"{b:12d} " + " ".join(f"{r:26.4f}" for r in row))


if __name__ == "__main__":
    main()
