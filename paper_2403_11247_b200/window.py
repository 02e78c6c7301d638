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
               pipelined=True, batched=False, chain_views=False):
    """WindowStep over a RenderStep: `views[i]` is keyframe i's world->camera view.

    pipelined: the rank's keyframes alternate between two view slots
    (RenderStep.view_slot) on two streams -- keyframe q+1's projection, binning
    and forward run while keyframe q's backward accumulates.  The backwards
    (and their read-modify-write of the shared gradient buffer) stay in order on
    one stream, so the result equals the sequential loop's up to the
    nondeterministic order of the backward's float atomics."""
    from . import csplat as cs

    if batched:
        return BatchedWindow(step, views, rank, world, group, reduce, chain_views=chain_views)
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


class BatchedWindow(WindowStep):
    """The rank's keyframes with ONE multi-view front (SURVEY §8(e)
    "multi-view projection that reads each Gaussian once"): per iteration

        prune + R-VQ (once) -> csplat_project_bin_views (every local keyframe's
        projection from one read and decode of each Gaussian, per-view tile
        buckets, one batched per-tile sort over all the keyframes) -> per
        keyframe csplat_render_fwd (front stream) and csplat_render_bwd with
        ACCUMULATE (back stream, in keyframe order: the chain's gradient
        read-modify-write) over two image / workspace slots -> all-reduce.

    chain_views=True replaces the per-keyframe chains by one
    csplat_chain_views over all keyframes (SKIP_CHAIN backwards into per-
    keyframe accumulators); on C5 it measured slower (13.0 vs 12.7 ms: nearly
    every warp of the face-ordered map has a visible lane in most views, so the
    per-view chain work is not saved and the one kernel is latency-bound).
    Memory per local keyframe: records 64 n B, counts 4 n B, its pair list and
    binning workspace (+ 48 n B accumulator with chain_views)."""

    def __init__(self, step, views, rank=None, world=None, group=None, reduce=True,
                 chain_views=False):
        from . import csplat as cs
        super().__init__(len(views), step.grads["flat"], None, step.prepare, rank, world, group,
                         reduce)
        self.st = step
        self.views = views
        dev = step.dev
        n, V = step.n, len(self.local)
        self.lviews = [views[k] for k in self.local]
        self.vb = cs.alloc_views(n, V, step.capacity, step.cam, dev)
        self.chain_views = chain_views
        wsb = cs.workspace_bytes(cs.OP_RENDER_BWD, n)   # a multiple of 256
        self.acc = torch.zeros((V if chain_views else 2, wsb), dtype=torch.uint8, device=dev)
        self.pose = torch.zeros((V, 6), device=dev)
        self.imgs = [{k: torch.empty_like(v) for k, v in step.img.items()} for _ in range(2)]
        self.s_front = torch.cuda.Stream(device=dev)
        self.s_back = torch.cuda.Stream(device=dev)
        self.front_done = [torch.cuda.Event() for _ in range(2)]
        self.slot_free = [torch.cuda.Event() for _ in range(2)]
        self.ups = None  # per-keyframe upstream (d_color, d_depth, d_sil); default: step's

    def check_capacity(self):
        """Pair capacity over every local keyframe since the last check (the views'
        status slots, one host read): raises on any overflow."""
        from . import csplat as cs
        st = self.vb["tile_range"][:, -1].cpu()
        self.vb["tile_range"][:, -1].zero_()
        worst = int(st[:, 1].numpy().view("uint32").max()) if len(st) else 0
        if int(st[:, 0].numpy().view("uint32").max() if len(st) else 0) & cs.STATUS_CAPACITY \
                or worst > self.vb["capacity"]:
            raise cs.CsplatError(f"{worst} pairs exceed the capacity {self.vb['capacity']}")
        return worst

    def run(self):
        from . import csplat as cs
        st = self.st
        main = torch.cuda.current_stream(self.flat.device)
        self.flat.zero_()
        self.pose.zero_()  # the per-keyframe backwards ACCUMULATE their pose gradients
        self.prepare_fn()
        g, vb = st.pruned, self.vb
        cs.project_bin_views(g, st.cam, self.lviews, vb, st.prm, st.cb)
        self.s_front.wait_stream(main)
        self.s_back.wait_stream(main)
        for q in range(len(self.local)):
            b = q % 2
            img = self.imgs[b]
            dC, dD, dS = self.ups[q] if self.ups is not None else st.upstream
            with torch.cuda.stream(self.s_front):
                if q >= 2:  # keyframe q-2's backward has finished with this slot
                    self.s_front.wait_event(self.slot_free[b])
                cs.render_fwd(vb["rec"][q], vb["pair_gid"][q], vb["tile_range"][q], st.cam,
                              st.prm, out=img)
                self.front_done[b].record(self.s_front)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[b])
                if self.chain_views:
                    cs.render_bwd(g, st.cam, self.lviews[q], vb["rec"][q], vb["pair_gid"][q],
                                  vb["tile_range"][q], img["t_final"], img["n_contrib"], dC, dD,
                                  dS, st.prm, st.cb, cs.SKIP_CHAIN | cs.WS_ZEROED,
                                  grads=st.grads, ws=self.acc[q])
                else:
                    grads = dict(st.grads, pose=self.pose[q])
                    cs.render_bwd(g, st.cam, self.lviews[q], vb["rec"][q], vb["pair_gid"][q],
                                  vb["tile_range"][q], img["t_final"], img["n_contrib"], dC, dD,
                                  dS, st.prm, st.cb, cs.ACCUMULATE, grads=grads, ws=self.acc[b])
                self.slot_free[b].record(self.s_back)
        main.wait_stream(self.s_front)
        main.wait_stream(self.s_back)
        if self.chain_views:
            cs.chain_views(g, st.cam, self.lviews, vb["rec"], self.acc, st.grads, pose=self.pose,
                           prm=st.prm, cb=st.cb, flags=cs.WS_ZEROED)
        for q, k in enumerate(self.local):
            self.poses[k] = self.pose[q]
        if self.world > 1 and self.reduce:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        return self.flat
