"""One rank of the DDP comm-hook check (tests/test_gpu_nccl.py): a small MLP
under DistributedDataParallel with the libesp hook.  (1) NONE/Allreduce gives
the gradients of DDP's own allreduce within fp32 tolerance; (2) DGC/Allgather
gives, bit for bit, the oracle's n-rank simulation of every parameter's local
gradients (the oracle's inputs are the ranks' local gradients, computed by a
non-DDP replica and all-gathered on the host -- never a CUDA-path result)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import esp_oracle as O  # noqa: E402
from paper_2205_14465_b200 import ddp as D  # noqa: E402
from torch.nn.parallel import DistributedDataParallel as DDP  # noqa: E402


def make_model():
    torch.manual_seed(1234)
    return torch.nn.Sequential(torch.nn.Linear(64, 300), torch.nn.ReLU(), torch.nn.Linear(300, 333),
                               torch.nn.ReLU(), torch.nn.Linear(333, 10)).cuda()


def batch(rank, step):
    g = torch.Generator().manual_seed(1000 * step + rank)
    return torch.randn(32, 64, generator=g).cuda(), torch.randint(0, 10, (32,), generator=g).cuda()


def grads_of(model):
    return [p.grad.detach().float().cpu().numpy().copy() for p in model.parameters()]


def local_grads(rank, step, sd):
    m = make_model()
    m.load_state_dict(sd)
    x, y = batch(rank, step)
    torch.nn.functional.cross_entropy(m(x), y).backward()
    return grads_of(m)


def main():
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))

    # (1) NONE / Allreduce == DDP's allreduce
    ref = DDP(make_model(), bucket_cap_mb=0.25)
    hk = DDP(make_model(), bucket_cap_mb=0.25)
    st = D.EspressoState(hk.module, lambda N: ("none", 1.0, "allreduce"))
    hk.register_comm_hook(st, D.espresso_hook)
    for m in (ref, hk):
        x, y = batch(rank, 0)
        torch.nn.functional.cross_entropy(m(x), y).backward()
    torch.cuda.synchronize()
    for a, b in zip(grads_of(ref.module), grads_of(hk.module)):
        np.testing.assert_allclose(b, a, rtol=1e-5, atol=1e-7)
    st.destroy()

    # (2) DGC 5% / Allgather, 2 steps, against the oracle
    model = DDP(make_model(), bucket_cap_mb=0.25)
    st = D.EspressoState(model.module, lambda N: ("dgc", 0.05, "allgather"))
    model.register_comm_hook(st, D.espresso_hook)
    cfg = O.Cfg("dgc", 0.05)
    params = list(model.module.parameters())
    states = [O.new_states(n, p.numel(), "allgather", cfg) for p in params]
    sd = {k: v.clone() for k, v in model.module.state_dict().items()}
    for step in range(2):
        for p in params:
            p.grad = None
        x, y = batch(rank, step)
        torch.nn.functional.cross_entropy(model(x), y).backward()
        torch.cuda.synchronize()
        got = grads_of(model.module)
        mine = np.concatenate([g.ravel() for g in local_grads(rank, step, sd)])
        allg = [torch.zeros(mine.size) for _ in range(n)]
        dist.all_gather_object(allg, mine)
        off = 0
        for i, p in enumerate(params):
            N = p.numel()
            per_rank = [np.asarray(allg[r][off:off + N], np.float32) for r in range(n)]
            off += N
            res = O.sync("allgather", cfg, per_rank, states[i], tensor_id=i)
            exp = res.outs[rank].reshape(got[i].shape)
            assert np.array_equal(got[i].view(np.uint32), exp.view(np.uint32)), f"param {i} step {step}"
    st.destroy()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}: ddp hook ok", flush=True)


if __name__ == "__main__":
    main()
