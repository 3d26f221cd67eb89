"""Debug: one fused (kind, routine, process) pair in an NCCL world, step by step."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import esp_oracle as O
from paper_2205_14465_b200 import esp as E
from synth.values import gradient
kind, routine, proc = sys.argv[1], sys.argv[2], int(sys.argv[3])
rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
w = E.World.nccl(rank)
N = 30_011
ctx = E.Ctx(w, kind, routine, N, tensor_id=5, ratio=0.02, process=proc)
cfg = O.Cfg(kind, 0.02, process=proc)
st = O.new_states(n, N, routine, cfg)
for s in range(3):
    grads = [gradient(N, step=s, rank=r, tensor=5) for r in range(n)]
    ref = O.sync(routine, cfg, grads, st, tensor_id=5)
    g = torch.from_numpy(grads[rank].copy()).cuda()
    print(f"rank {rank} step {s} start", flush=True)
    E.esp_sync(w, ctx, g)
    torch.cuda.synchronize()
    got = g.cpu().numpy()
    bad = np.nonzero(got.view(np.uint32) != ref.outs[rank].view(np.uint32))[0]
    print(f"rank {rank} step {s}: {bad.size} mismatches", flush=True)
print(f"rank {rank} done", flush=True)
