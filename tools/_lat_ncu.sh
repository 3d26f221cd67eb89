#!/bin/bash
mkdir -p gpurun_out/lat
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/lat1.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2205_14465_b200 import esp as E
torch.cuda.set_device(0)
w = E.World.nccl_single(0); sim = E.World.sim(2, 0)
c = E.Ctx(w, "dgc", "allgather", 256, ratio=0.01)
g = torch.randn(256, device="cuda"); pay = torch.empty(c.payload_bytes, dtype=torch.uint8, device="cuda")
for _ in range(5): E.esp_compress(c, g, pay)
c1 = E.Ctx(sim, "dgc", "allgather", 1 << 20, ratio=0.01)
g1 = torch.randn(2 << 20, device="cuda")
for _ in range(5): E.esp_sync(sim, c1, g1)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat/l.csv python /tmp/lat1.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/lat/l.csv")))
h=None
for r in rows:
    if r and r[0]=="ID": h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d["ID"], d["Kernel Name"].split("(")[0][:40], d["Grid Size"] if "Grid Size" in d else "", d["Metric Value"])
PY
