import torch, sys, time
sys.path.insert(0, '.')
from paper_2205_14465_b200 import esp as E
torch.cuda.set_device(0)
w = E.World.nccl_single(0)
for n in [1 << 12, 1 << 16, 1 << 19, 1 << 22]:
    for ratio in [0.01, 0.001]:
        c = E.Ctx(w, "dgc", "allgather", n, ratio=ratio)
        g = torch.randn(n, device="cuda") * 1e-2
        p = torch.empty(c.payload_bytes, dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(30):
            torch.cuda.synchronize(); t = time.perf_counter()
            E.esp_compress(c, g, p); torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e6)
        print(n, ratio, [round(x) for x in ts[:6]], round(sum(ts[10:]) / 20), file=sys.stderr)
        c.destroy()
