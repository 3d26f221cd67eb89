"""One big tensor through esp_compress (debug aid): python tools/dbg_big.py KIND RATIO LOG2_ELEMS"""
import sys
import torch
sys.path.insert(0, '.')
from paper_2205_14465_b200 import esp as E
kind, ratio, ex = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
torch.cuda.set_device(0)
w = E.World.nccl_single(0)
n = 1 << ex
c = E.Ctx(w, kind, "allgather", n, ratio=ratio)
g = torch.randn(n, device="cuda") * 1e-2
p = torch.empty(c.payload_bytes, dtype=torch.uint8, device="cuda")
for i in range(4):
    E.esp_compress(c, g, p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(5):
    E.esp_compress(c, g, p)
e1.record()
torch.cuda.synchronize()
print(kind, ratio, ex, "us per call", e0.elapsed_time(e1) / 5 * 1e3)
