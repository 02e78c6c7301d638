"""NEXT-4: random-ray global bundle adjustment (Sec 3.4; reading R30).

"We randomly sample a total number of N rays from our global keyframe database
to optimize our scene representation as well as camera poses.  This phase
optimizes a loss similar to tracking loss, and we also add an SSIM loss to RGB
rendering."  The N rays are N/64 random 8x8 patches (the SSIM window), drawn
over all keyframes (``scenes.synth.sample_patches``).  One BA iteration:

    prepare the map (mask prune + R-VQ assignment, once)
    per local keyframe:  csplat_ba_patches   -> active-tile mask, |R| share
    [ranks > 1: SUM all-reduce of the 8-byte |R|: the Eq 12 normaliser is
     sample-wide]
    per local keyframe with patches:
        project -> csplat_bin_tiles_active (only the sampled tiles)
        -> render_fwd -> csplat_ba_patch_loss -> render_bwd(ACCUMULATE, own pose)
    [ranks > 1: SUM all-reduce of the flat Gaussian gradient and the loss]

Keyframes are sharded round-robin over ranks exactly as the mapping window
(``window.shard``); poses stay rank-local.  Every stage is a libcsplat kernel;
the loop, the sharding and the collectives are host plumbing.  The GPU backend
is injected as in ``window.WindowStep`` so the gloo tests exercise the
sharding and the two reductions without a GPU.
"""
from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from .window import shard


class BAStep:
    def __init__(self, n_keyframes: int, flat_grad: torch.Tensor, n_valid: torch.Tensor,
                 loss3: torch.Tensor, count_fn: Callable[[int], None],
                 render_fn: Callable[[int, torch.Tensor], None],
                 prepare_fn: Callable[[], None] | None = None, rank: int | None = None,
                 world: int | None = None, group=None):
        self.world = world if world is not None else (dist.get_world_size(group)
                                                      if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group)
                                                   if dist.is_initialized() else 0)
        self.group = group
        self.local = shard(n_keyframes, self.rank, self.world)
        self.flat, self.n_valid, self.loss3 = flat_grad, n_valid, loss3
        self.count_fn, self.render_fn, self.prepare_fn = count_fn, render_fn, prepare_fn
        self.poses = {k: torch.zeros(6, dtype=flat_grad.dtype, device=flat_grad.device)
                      for k in self.local}

    def run(self):
        """One BA iteration; returns the (all-reduced) flat gradient buffer."""
        self.flat.zero_()
        self.n_valid.zero_()
        self.loss3.zero_()
        if self.prepare_fn is not None:
            self.prepare_fn()
        for k in self.local:
            self.count_fn(k)
        if self.world > 1:
            dist.all_reduce(self.n_valid, op=dist.ReduceOp.SUM, group=self.group)
        if getattr(self, "pipe", None) is None:
            for k in self.local:
                self.poses[k].zero_()
                self.render_fn(k, self.poses[k])
        else:  # two view slots on two streams: keyframe q+1's front under q's backward
            front_fn, back_fn, s_front, s_back, front_done, slot_free = self.pipe
            main = torch.cuda.current_stream(self.flat.device)
            s_front.wait_stream(main)
            s_back.wait_stream(main)
            for q, k in enumerate(self.local):
                b = q % 2
                with torch.cuda.stream(s_front):
                    if q >= 2:
                        s_front.wait_event(slot_free[b])
                    front_fn(k, b)
                    front_done[b].record(s_front)
                with torch.cuda.stream(s_back):
                    s_back.wait_event(front_done[b])
                    self.poses[k].zero_()
                    back_fn(k, b, self.poses[k])
                    slot_free[b].record(s_back)
            main.wait_stream(s_front)
            main.wait_stream(s_back)
        if self.world > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
            dist.all_reduce(self.loss3, op=dist.ReduceOp.SUM, group=self.group)
        return self.flat


def ba_loss_value(loss3, lambda_depth=1.0, lambda_ssim=0.2) -> float:
    """L_ba = L_c + lambda_d L_d + lambda_s (1 - SSIM) from the reduced shares."""
    l = [float(x) for x in loss3]
    return l[0] + lambda_depth * l[1] + lambda_ssim * (1.0 - l[2])


def gpu_ba(step, views, obs_color, obs_depth, patches, lambda_depth=1.0, lambda_ssim=0.2,
           rank=None, world=None, group=None, pipelined=True):
    """BAStep over a RenderStep: keyframe k has view `views[k]`, observed images
    obs_color[k] [3,H,W] / obs_depth[k] [H,W] (device; only local keyframes are
    read) and patch ids `patches[k]` (int32, see scenes.synth.sample_patches)."""
    from . import csplat as cs

    dev = step.dev
    n_rays = 64 * sum(int(len(p)) for p in patches)
    n_valid = torch.zeros(1, dtype=torch.int64, device=dev)
    loss3 = torch.zeros(3, dtype=torch.float32, device=dev)
    up = (torch.empty_like(step.img["color"]), torch.empty_like(step.img["depth"]),
          torch.empty_like(step.img["sil"]))
    words = cs.tile_mask_words(step.cam)
    pt, masks = {}, {}

    def count(k):
        if k not in pt:
            pt[k] = torch.as_tensor(patches[k], dtype=torch.int32).to(dev)
            masks[k] = torch.empty(words, dtype=torch.int32, device=dev)
        cs.ba_patches(obs_depth[k], step.cam, pt[k], tile_active=masks[k], n_valid=n_valid)

    def render(k, pose):
        if pt[k].numel() == 0:
            return
        step.project_bin(views[k], tile_active=masks[k])
        step.forward()
        cs.ba_patch_loss(step.img, obs_color[k], obs_depth[k], step.cam, pt[k], n_rays, n_valid,
                         lambda_depth, lambda_ssim, out=up, loss3=loss3)
        step.set_upstream(*up)
        step.backward(views[k], flags=cs.ACCUMULATE, pose=pose)

    ba = BAStep(len(views), step.grads["flat"], n_valid, loss3, count, render, step.prepare,
                rank, world, group)
    ba.n_rays = n_rays
    ba.pipe = None
    slots = [step]
    # pair capacity over every keyframe since the last check (all view slots'
    # status words, one host read; pipeline.RenderStep.check_capacity)
    ba.check_capacity = lambda: slots[0].check_capacity(slots[1:])
    if pipelined:  # window.py's two-slot pipeline: per-slot buffers and upstream
        slots.append(step.view_slot())
        ups = [up, tuple(torch.empty_like(t) for t in up)]

        def front(k, b):
            if pt[k].numel() == 0:
                return
            sl = slots[b]
            sl.project_bin(views[k], tile_active=masks[k])
            sl.forward()
            cs.ba_patch_loss(sl.img, obs_color[k], obs_depth[k], sl.cam, pt[k], n_rays, n_valid,
                             lambda_depth, lambda_ssim, out=ups[b], loss3=loss3)

        def back(k, b, pose):
            if pt[k].numel() == 0:
                return
            sl = slots[b]
            sl.set_upstream(*ups[b])
            sl.backward(views[k], flags=cs.ACCUMULATE, pose=pose)

        ba.pipe = (front, back, torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev),
                   [torch.cuda.Event() for _ in range(2)], [torch.cuda.Event() for _ in range(2)])
    return ba


class BatchedBA:
    """NEXT-4 with the sparse views batched (the rank's keyframes through one
    multi-view front): per iteration

        prune + R-VQ -> every keyframe's patch mask and valid-ray count
        (csplat_ba_patches) -> csplat_project_bin_views with per-keyframe tile
        masks AND tile lists (one projection read per Gaussian for all
        keyframes; only the sampled tiles are bucketed and sorted) -> per
        keyframe csplat_render_fwd_list (the sampled tiles only), the patch
        loss, csplat_render_bwd_list (SKIP_CHAIN | WS_ZEROED into the
        keyframe's own accumulator) -> csplat_chain_views over all keyframes
        (few Gaussians per view are reached) -> all-reduce.

    Same results as gpu_ba (tests); the tile lists come from the host-side
    patch sample (the method's random draw, an input)."""

    def __init__(self, step, views, obs_color, obs_depth, patches, lambda_depth=1.0,
                 lambda_ssim=0.2, rank=None, world=None, group=None):
        from . import csplat as cs
        self.world = world if world is not None else (dist.get_world_size(group)
                                                      if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group)
                                                   if dist.is_initialized() else 0)
        self.group = group
        self.local = shard(len(views), self.rank, self.world)
        self.st, dev = step, step.dev
        self.flat = step.grads["flat"]
        self.n_valid = torch.zeros(1, dtype=torch.int64, device=dev)
        self.loss3 = torch.zeros(3, dtype=torch.float32, device=dev)
        self.n_rays = 64 * sum(int(len(p)) for p in patches)
        self.lam = (lambda_depth, lambda_ssim)
        self.lviews = [views[k] for k in self.local]
        self.obs = [(obs_color[k], obs_depth[k]) for k in self.local]
        cam = step.cam
        tx, _ = cs.tiles(cam)
        bw = cam["width"] // 8
        V = len(self.local)
        lists = []
        for k in self.local:
            p = np.asarray(patches[k], dtype=np.int64)
            by, bx = p // bw, p % bw
            lists.append(np.unique((by * 8 // 16) * tx + (bx * 8 // 16)))
        self.max_list = max([len(t) for t in lists] + [1])
        tl = np.zeros((V, 1 + self.max_list), dtype=np.int32)
        for q, t in enumerate(lists):
            tl[q, 0] = len(t)
            tl[q, 1:1 + len(t)] = t
        self.tile_lists = torch.tensor(tl, device=dev)
        self.pt = [torch.as_tensor(patches[k], dtype=torch.int32).to(dev) for k in self.local]
        self.masks = torch.zeros((V, cs.tile_mask_words(cam)), dtype=torch.int32, device=dev)
        self.vb = cs.alloc_views(step.n, V, step.capacity, cam, dev)
        wsb = cs.workspace_bytes(cs.OP_RENDER_BWD, step.n)
        self.acc = torch.zeros((V, wsb), dtype=torch.uint8, device=dev)
        self.pose = torch.zeros((V, 6), device=dev)
        self.poses = {k: self.pose[q] for q, k in enumerate(self.local)}
        self.imgs = [{k: torch.empty_like(v) for k, v in step.img.items()} for _ in range(2)]
        self.ups = [(torch.empty_like(step.img["color"]), torch.empty_like(step.img["depth"]),
                     torch.empty_like(step.img["sil"])) for _ in range(2)]
        self.s_front = torch.cuda.Stream(device=dev)
        self.s_back = torch.cuda.Stream(device=dev)
        self.front_done = [torch.cuda.Event() for _ in range(2)]
        self.slot_free = [torch.cuda.Event() for _ in range(2)]

    def check_capacity(self):
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
        st, vb = self.st, self.vb
        main = torch.cuda.current_stream(self.flat.device)
        self.flat.zero_()
        self.n_valid.zero_()
        self.loss3.zero_()
        st.prepare()
        g = st.pruned
        for q in range(len(self.local)):
            cs.ba_patches(self.obs[q][1], st.cam, self.pt[q], tile_active=self.masks[q],
                          n_valid=self.n_valid)
        if self.world > 1:
            dist.all_reduce(self.n_valid, op=dist.ReduceOp.SUM, group=self.group)
        cs.project_bin_views(g, st.cam, self.lviews, vb, st.prm, st.cb, tile_active=self.masks,
                             tile_lists=self.tile_lists, max_list=self.max_list)
        self.s_front.wait_stream(main)
        self.s_back.wait_stream(main)
        for q in range(len(self.local)):
            b = q % 2
            img, up = self.imgs[b], self.ups[b]
            with torch.cuda.stream(self.s_front):
                if q >= 2:
                    self.s_front.wait_event(self.slot_free[b])
                if self.pt[q].numel():
                    cs.render_fwd(vb["rec"][q], vb["pair_gid"][q], vb["tile_range"][q], st.cam,
                                  st.prm, out=img, tile_list=self.tile_lists[q],
                                  max_tiles=self.max_list)
                    cs.ba_patch_loss(img, self.obs[q][0], self.obs[q][1], st.cam, self.pt[q],
                                     self.n_rays, self.n_valid, *self.lam, out=up,
                                     loss3=self.loss3)
                self.front_done[b].record(self.s_front)
            with torch.cuda.stream(self.s_back):
                self.s_back.wait_event(self.front_done[b])
                if self.pt[q].numel():
                    cs.render_bwd(g, st.cam, self.lviews[q], vb["rec"][q], vb["pair_gid"][q],
                                  vb["tile_range"][q], img["t_final"], img["n_contrib"], *up,
                                  st.prm, st.cb, cs.SKIP_CHAIN | cs.WS_ZEROED, grads=st.grads,
                                  ws=self.acc[q], tile_list=self.tile_lists[q],
                                  max_tiles=self.max_list)
                self.slot_free[b].record(self.s_back)
        main.wait_stream(self.s_front)
        main.wait_stream(self.s_back)
        cs.chain_views(g, st.cam, self.lviews, vb["rec"], self.acc, st.grads, pose=self.pose,
                       prm=st.prm, cb=st.cb, flags=cs.WS_ZEROED)
        if self.world > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
            dist.all_reduce(self.loss3, op=dist.ReduceOp.SUM, group=self.group)
        return self.flat
