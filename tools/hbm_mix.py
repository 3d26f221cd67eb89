"""Calibrate achievable HBM bandwidth on this GPU for the access mixes of the
hot path: copy (1R:1W), add (2R:1W, the h1 streaming pass), fill (write only,
the h2 output), sum (read only).  torch kernels, CUDA events, best of 20."""
import json

import torch

N = 1 << 28
a = torch.randn(N, device="cuda")
b = torch.randn(N, device="cuda")
c = torch.empty(N, device="cuda")


def bw(fn, nbytes, reps=20):
    best = 1e9
    for _ in range(3):
        fn()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / (best / 1e3) / 1e9


out = {
    "copy_1r1w": bw(lambda: c.copy_(a), 8 * N),
    "add_2r1w": bw(lambda: torch.add(a, b, out=c), 12 * N),
    "inplace_add_2r1w": bw(lambda: a.add_(b), 12 * N),
    "fill_1w": bw(lambda: c.fill_(0.5), 4 * N),
    "sum_1r": bw(lambda: a.sum(), 4 * N),
}
print(json.dumps(out))
