"""Keyframe-window data parallelism (north_star "the mapping
and global-BA keyframe window").

Every rank holds a full replica of the Gaussian map and renders the keyframes
{i : i mod G = rank} of the window (fwd + bwd, gradients ACCUMULATEd into one
flat fp32 buffer of 15 planes).  The one exchange of an iteration is a SUM
all-reduce of that buffer (torch.distributed / NCCL over NVLink on GPUs, gloo
in the CPU tests).  Per-keyframe pose gradients stay on the rank that owns the
keyframe -- no collective for them.  Because every rank receives the identical
reduced buffer, a deterministic update keeps the replicas bit-identical.

The render backend is injected (``render_fn(kf, grads, pose)``): on a GPU it
is ``RenderStep.render`` (libcsplat kernels); the gloo tests use a host stub,
so the sharding/reduction logic is exercised without a GPU.
"""
from __future__ import annotations

from typing import Callable, Sequence

import torch
import torch.distributed as dist


def shard(n_keyframes: int, rank: int, world: int) -> list[int]:
    """Round-robin keyframe ownership: keyframe i -> rank i mod world."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return list(range(rank, n_keyframes, world))


class WindowStep:
    def __init__(self, n_keyframes: int, flat_grad: torch.Tensor,
                 render_fn: Callable[[int, torch.Tensor], None],
                 prepare_fn: Callable[[], None] | None = None, rank: int | None = None,
                 world: int | None = None, group=None, reduce: bool = True):
        self.world = world if world is not None else (dist.get_world_size(group)
                                                      if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group)
                                                   if dist.is_initialized() else 0)
        self.group = group
        self.reduce = reduce  # False: the caller issues the all-reduce (e.g. outside a graph)
        self.local = shard(n_keyframes, self.rank, self.world)
        self.flat = flat_grad
        self.render_fn = render_fn
        self.prepare_fn = prepare_fn
        self.poses = {k: torch.zeros(6, dtype=flat_grad.dtype, device=flat_grad.device)
                      for k in self.local}

    def run(self):
        """One window iteration: local renders accumulate, then one all-reduce."""
        self.flat.zero_()
        if self.prepare_fn is not None:
            self.prepare_fn()
        for k in self.local:
            self.poses[k].zero_()
            self.render_fn(k, self.poses[k])
        if self.world > 1 and self.reduce:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        return self.flat


def apply_sgd(params: Sequence[torch.Tensor], grads: Sequence[torch.Tensor], lr: float):
    """A deterministic replicated update (identical on every rank)."""
    with torch.no_grad():
        for p, g in zip(params, grads):
            p.sub_(lr * g)


def gpu_window(step, views, rank=None, world=None, group=None, reduce=True,
               pipelined=True):
    """WindowStep over a RenderStep: `views[i]` is keyframe i's world->camera view.

    pipelined: the rank's keyframes alternate between two view slots
    (RenderStep.view_slot) on two streams -- keyframe q+1's projection, binning
    and forward run while keyframe q's backward accumulates.  The backwards
    (and their read-modify-write of the shared gradient buffer) stay in order on
    one stream, so the result equals the sequential loop's up to the
    nondeterministic order of the backward's float atomics."""
    from . import csplat as cs

    if not pipelined:
        def render(k, pose):
            step.render(views[k], flags=cs.ACCUMULATE, pose=pose)

        return WindowStep(len(views), step.grads["flat"], render, step.prepare, rank, world,
                          group, reduce)
    return PipelinedWindow(step, views, rank, world, group, reduce)


class PipelinedWindow(WindowStep):
    """WindowStep whose local renders are software-pipelined over two view slots."""

    def check_capacity(self):
        """Pair capacity over every keyframe rendered since the last check (both
        view slots' status words; one host read): raises on any overflow."""
        return self.slots[0].check_capacity(self.slots[1:])

    def __init__(self, step, views, rank=None, world=None, group=None, reduce=True):
        super().__init__(len(views), step.grads["flat"], None, step.prepare, rank, world, group,
                         reduce)
        self.views = views
        self.slots = [step, step.view_slot()]
        dev = step.dev
        self.s_front = torch.cuda.Stream(device=dev)
        self.s_back = torch.cuda.Stream(device=dev)
        self.front_done = [torch.cuda.Event() for _ in range(2)]
        self.slot_free = [torch.cuda.Event() for _ in range(2)]

    def run(self):
        from . import csplat as cs
        main = torch.cuda.current_stream(self.flat.device)
        self.flat.zero_()
        self.prepare_fn()
        self.s_front.wait_stream(main)
        self.s_back.wait_stream(main)
        for q, k in enumerate(self.local):
            b = q % 2
            sl = self.slots[b]
            with torch.cuda.stream(self.s_front):
                if q >= 2:  # keyframe q-2's backward has finished with this slot
                    self.s_front.wait_event(self.slot_free[b])
                sl.project_bin_forward(self.views[k])
                self.front_done[b].record(self.s_front)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[b])
                self.poses[k].zero_()
                sl.backward(self.views[k], cs.ACCUMULATE, self.poses[k])
                self.slot_free[b].record(self.s_back)
        main.wait_stream(self.s_front)
        main.wait_stream(self.s_back)
        if self.world > 1 and self.reduce:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        return self.flat
