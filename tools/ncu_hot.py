"""Summarise an ncu source page (SASS) for one kernel: top stalled instructions
and the stall-reason totals.  usage: ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
import re
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = [b for b in out.split('"Kernel Name"')[1:] if re.search(kre, b.split("\n", 1)[0])]
for blk in blocks[:1]:
    lines = blk.split("\n", 1)
    print("kernel:", lines[0][:120])
    rows = list(csv.reader(io.StringIO(lines[1])))
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    S = ci["Warp Stall Sampling (All Samples)"]
    tot = sum(float(r[S] or 0) for r in data)
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {h: sum(float(r[ci[h]] or 0) for r in data) for h in stalls}
    print("samples", tot)
    print("stalls:", ", ".join(f"{k[6:]}={v / tot:.0%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    data.sort(key=lambda r: -float(r[S] or 0))
    for r in data[:top]:
        det = [f"{k[6:]}:{int(float(r[ci[k]]))}" for k in stalls if float(r[ci[k]] or 0) > 0.15 * float(r[S] or 1)]
        print(f"{float(r[S]) / tot:6.1%} {r[ci['Address']][-5:]} {r[ci['Source']].strip()[:70]:70s} {' '.join(det)}")
