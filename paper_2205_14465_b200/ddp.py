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
        self.layout: dict[int, tuple] = {}   # bucket index -> its parameters' ids

    def note_bucket(self, index: int, ids: tuple):
        """DDP rebuilds its buckets after the first iteration (and may again, e.g.
        with find_unused_parameters): when a bucket's parameter list changes,
        the cached libesp plans of the old lists are freed on every rank (every
        rank sees the same rebuild at the same step)."""
        old = self.layout.get(index)
        if old is not None and old != ids:
            self.world.drop_plans()
            self.layout.clear()
        self.layout[index] = ids

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
    if bucket.buffer().dtype != torch.float32:
        raise TypeError(f"espresso_hook synchronises fp32 gradients; got a {bucket.buffer().dtype} bucket "
                        "(keep fp32 master gradients or cast before the hook)")
    state.note_bucket(bucket.index(), tuple(state.pid[id(p)] for p in params))
    ctxs = [state.ctx(p, g.numel()) for p, g in zip(params, grads)]
    E.esp_sync_many(state.world, ctxs, grads, torch.cuda.current_stream())
    fut = torch.futures.Future()
    fut.set_result(bucket.buffer())
    return fut
