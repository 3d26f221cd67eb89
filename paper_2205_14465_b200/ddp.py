"""DDP communication hook that synchronises gradient buckets with libesp
(training integration).

PyTorch DDP hands every gradient bucket to the hook as soon as its gradients
are ready during the backward pass, so compression of early buckets overlaps
the backward computation of later layers -- the wait-free back-propagation
overlap the paper builds on.  The hook runs the per-tensor compression
strategy (the paper's option c_j per tensor) on the bucket's
per-parameter gradient views with one esp_sync_many call (h1 -> routine -> h2,
all in libesp's kernels on the current stream) and returns the bucket buffer,
which then holds the aggregated (MEAN) gradients.  No arithmetic happens here:
this module only maps parameters to libesp contexts.

    state = EspressoState(model, rule)      # rule(numel) -> (kind, ratio, routine[, extra])
    ddp.register_comm_hook(state, espresso_hook)
"""
import torch

from . import esp as E


class EspressoState:
    """One libesp world over the default process group and one context (EF
    state) per parameter; tensor ids are the parameters' positions in
    model.parameters(), identical on every rank."""

    def __init__(self, model: torch.nn.Module, rule, world: E.World | None = None):
        self.world = world if world is not None else E.World.nccl(torch.cuda.current_device())
        self.rule = rule
        self.pid = {id(p): i for i, p in enumerate(model.parameters())}
        self.ctxs: dict[int, E.Ctx] = {}

    def ctx(self, p: torch.Tensor, numel: int) -> E.Ctx:
        i = self.pid[id(p)]
        c = self.ctxs.get(i)
        if c is None:
            kind, ratio, routine, *extra = self.rule(numel)
            c = E.Ctx(self.world, kind, routine, numel, tensor_id=i, ratio=ratio, **(extra[0] if extra else {}))
            self.ctxs[i] = c
        return c

    def destroy(self):
        for c in self.ctxs.values():
            c.destroy()
        self.ctxs.clear()
        self.world.destroy()


def espresso_hook(state: EspressoState, bucket: torch.distributed.GradBucket) -> torch.futures.Future[torch.Tensor]:
    grads = bucket.gradients()
    params = bucket.parameters()
    ctxs = [state.ctx(p, g.numel()) for p, g in zip(params, grads)]
    E.esp_sync_many(state.world, ctxs, grads, torch.cuda.current_stream())
    fut = torch.futures.Future()
    fut.set_result(bucket.buffer())
    return fut
