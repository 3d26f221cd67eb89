"""Per-CUDA-line warp-stall samples and executed instructions of one kernel
from `ncu -i REP --page source --csv --print-source cuda,sass` output.
usage: ncu_lines.py CSV [ctas] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ctas = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = next(r for r in rows if r and r[0] == "Line No")
c = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
stc = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not" not in h]
data, tot = [], {}
for r in rows:
    if len(r) > c and r[0] and r[0][0].isdigit():
        try:
            v = float(r[c])
        except ValueError:
            continue
        st = [(float(r[j]) if r[j] not in ("-", "") else 0.0, hdr[j][6:]) for j in stc]
        for a, b in st:
            tot[b] = tot.get(b, 0) + a
        data.append((v, int(r[0]), r[1][:80], sorted(st, reverse=True)[:2], float(r[ie] or 0)))
T = sum(d[0] for d in data)
print(f"samples {T:.0f}, warp instructions per CTA {sum(d[4] for d in data) / ctas:.0f}")
print("stalls:", [(k, int(v)) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]])
for v, l, s, st, n in sorted(data, reverse=True)[:top]:
    print(f"{v / T:6.1%} {n / ctas:7.0f} {l:5d} {s:80s} {[(b, int(a)) for a, b in st]}")
