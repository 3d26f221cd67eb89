"""Per-call fixed overheads on the user stream: zero-region memset and the
pinned H2D upload of the dynamic segment table (debug aid, not a test)."""
import torch

torch.cuda.set_device(0)
buf = torch.empty(10 << 20, dtype=torch.uint8, device="cuda")
h = torch.empty(6400, dtype=torch.uint8).pin_memory()
d = torch.empty(6400, dtype=torch.uint8, device="cuda")


def t(fn, n=50):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


print("memset 10MB us", t(lambda: buf.zero_()))
print("h2d 6.4KB us", t(lambda: d.copy_(h, non_blocking=True)))
print("both us", t(lambda: (buf.zero_(), d.copy_(h, non_blocking=True))))
