"""One pass of the whole hot path over one view,
with every buffer preallocated so the step can be replayed or captured in a
CUDA graph:

    mask_prune (a9, a1)  ->  rvq_assign scale + rotation (a2)
    -> project with R-VQ decode + mask (a1, a2, a3) -> bin_tiles (a4, a5)
    -> render_fwd (a6) -> render_bwd incl. chain, STE and pose (a7, a8)

Every stage is a libcsplat call (paper_2403_11247_b200.csplat); torch only
provides device memory and streams.  The survivor count of the prune stays on
the device (n_dev), so the step has no host synchronisation.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import csplat as cs


# csplat_project_bin (projection with the bucket pass fused in) on the step's
# path; CSPLAT_FUSED_BIN=0 selects the separate csplat_project + csplat_bin_tiles
FUSED_BIN = os.environ.get("CSPLAT_FUSED_BIN", "1") == "1"


def _on_device(v) -> bool:
    return isinstance(v, torch.Tensor) and v.is_cuda

class RenderStep:
    def __init__(self, planes: dict, cam: dict, codebook: dict | None, device="cuda",
                 prm: cs.Params | None = None, pair_capacity: int | None = None,
                 flags: int = 0):
        self.cam = dict(cam)
        self.prm = prm or cs.params()
        self.flags = flags
        self.dev = torch.device(device)
        self.g = cs.GaussianMap.from_numpy(planes, device=self.dev)
        n = self.n = self.g.n
        H, W = cam["height"], cam["width"]
        # a9 outputs (capacity n) and the device survivor count
        self.pruned = cs.GaussianMap(**{k: torch.empty_like(getattr(self.g, k)) for k in
                                        ("mean", "opacity", "rgb", "log_scale", "quat", "mask")})
        self.n_kept = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.keep_map = torch.empty(n, dtype=torch.int32, device=self.dev)
        self.ws_prune = torch.empty(cs.workspace_bytes(cs.OP_MASK_PRUNE, n), dtype=torch.uint8,
                                    device=self.dev)
        # a2 codebooks and indices
        self.codes = None
        if codebook is not None:
            sc = torch.as_tensor(codebook["scale_codes"], dtype=torch.float32).contiguous().to(self.dev)
            rc = torch.as_tensor(codebook["rot_codes"], dtype=torch.float32).contiguous().to(self.dev)
            L, P = sc.shape[:2]
            dt = torch.uint8 if P <= 256 else torch.int16
            self.cb = cs.CodebookT(sc, rc, torch.zeros((L, n), dtype=dt, device=self.dev),
                                   torch.zeros((L, n), dtype=dt, device=self.dev))
        else:
            self.cb = None
        # a3 outputs
        self.rec = torch.empty((n, 16), dtype=torch.int32, device=self.dev)
        self.count = torch.empty(n, dtype=torch.int32, device=self.dev)
        # a4/a5: size the pair buffers from a probe bin of this scene at the first view
        self.tile_range = cs.alloc_tile_range(cam, self.dev)
        self.n_pairs = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.capacity = pair_capacity or 1
        self._alloc_pairs(self.capacity)
        # a6 outputs
        self.img = dict(color=torch.empty((3, H, W), device=self.dev),
                        depth=torch.empty((H, W), device=self.dev),
                        sil=torch.empty((H, W), device=self.dev),
                        t_final=torch.empty((H, W), device=self.dev),
                        n_contrib=torch.empty((H, W), dtype=torch.int32, device=self.dev))
        # a7/a8
        self.grads = cs.alloc_grads(n, self.dev, pose_only=bool(flags & cs.POSE_ONLY))
        self.ws_bwd = torch.empty(cs.workspace_bytes(cs.OP_RENDER_BWD, n), dtype=torch.uint8,
                                  device=self.dev)
        self.upstream = None
        self.graph = None
        self.side = torch.cuda.Stream(device=self.dev)
        self.single_stream = os.environ.get("CSPLAT_SINGLE_STREAM", "0") == "1"

    def _alloc_pairs(self, cap):
        self.capacity = cap
        self.pair_gid = torch.empty(cap, dtype=torch.int32, device=self.dev)
        self.ws_bin = torch.empty(cs.workspace_bytes(cs.OP_BIN_TILES, self.n, cap, self.cam),
                                  dtype=torch.uint8, device=self.dev)

    def size_pairs(self, view, margin=1.25, views=()):
        """Size the pair buffers: run the front of the path once per given view
        (synchronously, into a generous probe buffer) and keep the worst count
        x margin -- shrinking the probe buffer again.  Returns the worst count."""
        worst = 0
        for v in [view, *views]:
            self.front(v, sync_probe=True)
            worst = max(worst, int(self.n_pairs.item()))
        self._alloc_pairs(int(worst * margin) + 4096)
        cs.clear_status(self.tile_range)
        return worst

    def view_slot(self):
        """A second set of per-view buffers (records, pairs, images, workspaces)
        over the SAME prepared map, codebook indices, upstream and gradient
        buffers: two slots let one view's projection / binning / forward run
        while the previous view's backward accumulates (window.py)."""
        import copy
        sl = copy.copy(self)
        n, dev = self.n, self.dev
        sl.rec = torch.empty_like(self.rec)
        sl.count = torch.empty_like(self.count)
        sl.tile_range = torch.zeros_like(self.tile_range)
        sl.n_pairs = torch.zeros_like(self.n_pairs)
        sl._alloc_pairs(self.capacity)
        sl.img = {k: torch.empty_like(v) for k, v in self.img.items()}
        sl.ws_bwd = torch.empty_like(self.ws_bwd)
        sl.graph = None
        assert sl.n == n and sl.dev == dev
        return sl

    def set_upstream(self, d_color, d_depth, d_sil):
        self.upstream = (d_color, d_depth, d_sil)

    # ---- stages -------------------------------------------------------------
    def prepare(self):
        """a9 (mask prune) -> a2 (R-VQ assignment of the survivors): once per
        iteration, shared by every view rendered from the same map."""
        self.prune()
        self.assign_codes()

    def prune(self):
        """a9: the codebook indices are re-assigned after, so only attribute planes
        are compacted."""
        cs.mask_prune(self.g, None, self.prm.mask_eps, float("nan"), out=self.pruned,
                      keep_map=self.keep_map, n_kept=self.n_kept, ws=self.ws_prune)

    def assign_codes(self):
        """a2 on the survivors (scale and rotation codebooks)."""
        g = self.pruned
        if self.cb is not None:
            # the scale and rotation assignments are independent: run them
            # concurrently (fork/join on a side stream; preserved by graph capture)
            main = torch.cuda.current_stream(self.dev)
            if self.single_stream:  # profilers serialise kernels: keep one stream
                cs.rvq_assign(g.log_scale, self.cb.scale_codes, n_dev=self.n_kept,
                              idx=self.cb.scale_idx, want_recon=False, stream=main)
                cs.rvq_assign(g.quat, self.cb.rot_codes, n_dev=self.n_kept,
                              idx=self.cb.rot_idx, want_recon=False, stream=main)
                return
            self.side.wait_stream(main)
            cs.rvq_assign(g.log_scale, self.cb.scale_codes, n_dev=self.n_kept,
                          idx=self.cb.scale_idx, want_recon=False, stream=main)
            cs.rvq_assign(g.quat, self.cb.rot_codes, n_dev=self.n_kept, idx=self.cb.rot_idx,
                          want_recon=False, stream=self.side)
            main.wait_stream(self.side)

    def render(self, view, flags=None, pose=None):
        """a3 -> a4/a5 -> a6 -> a7/a8 for one view of the prepared map."""
        self.project_bin_forward(view)
        self.backward(view, flags, pose)

    def front(self, view, sync_probe=False):
        """a9 -> a2 -> a3 -> a4/a5."""
        self.prepare()
        self.project_bin(view, sync_probe)

    def project_bin(self, view, sync_probe=False, tile_active=None):
        g = self.pruned
        if FUSED_BIN and not sync_probe:  # the bucket pass inside the projection kernel
            cs.project_bin(g, self.cam, view, self.capacity, self.prm, self.cb, rec=self.rec,
                           count=self.count, ws=self.ws_bin,
                           out=dict(pair_gid=self.pair_gid,
                                    tile_range=self.tile_range, n_pairs_dev=self.n_pairs),
                           sync=False, tile_active=tile_active)
            return
        cs.project(g, self.cam, view, self.prm, self.cb, rec=self.rec, count=self.count)
        if sync_probe:
            big = max(self.capacity, 64 * self.n + 4096)
            if big > self.capacity:
                self._alloc_pairs(big)
        cs.bin_tiles(self.rec, self.count, self.cam, self.capacity, ws=self.ws_bin,
                     out=dict(pair_gid=self.pair_gid,
                              tile_range=self.tile_range, n_pairs_dev=self.n_pairs),
                     sync=sync_probe, tile_active=tile_active)

    def forward(self):
        cs.render_fwd(self.rec, self.pair_gid, self.tile_range, self.cam, self.prm, out=self.img)

    def backward(self, view, flags=None, pose=None):
        dC, dD, dS = self.upstream
        grads = self.grads if pose is None else dict(self.grads, pose=pose)
        cs.render_bwd(self.pruned, self.cam, view, self.rec, self.pair_gid, self.tile_range,
                      self.img["t_final"], self.img["n_contrib"], dC, dD, dS, self.prm, self.cb,
                      self.flags if flags is None else flags, grads=grads, ws=self.ws_bwd)

    def step(self, view):
        self.prepare()
        self.render_view(view)

    def render_view(self, view):
        """a3 .. a8 of one view of the prepared map (no prune / R-VQ)."""
        if FUSED_BIN and not (self.flags & cs.POSE_ONLY) and not _on_device(view):
            # a3 .. a8 in one library call (per tile chunk: sort -> fwd -> bwd)
            dC, dD, dS = self.upstream
            cs.render_step(self.pruned, self.cam, view, self.capacity, dC, dD, dS, self.prm,
                           self.cb, self.flags, rec=self.rec, count=self.count, ws=self.ws_bin,
                           out=dict(pair_gid=self.pair_gid,
                                    tile_range=self.tile_range, n_pairs_dev=self.n_pairs),
                           img=self.img, grads=self.grads, ws_bwd=self.ws_bwd)
            return
        self.project_bin_forward(view)
        self.backward(view)

    def project_bin_forward(self, view):
        """a3 -> a4/a5 -> a6: one csplat_project_bin_render call (the per-tile
        sort and the forward pipelined in tile chunks) unless CSPLAT_FUSED_BIN=0."""
        if FUSED_BIN:
            cs.project_bin_render(self.pruned, self.cam, view, self.capacity, self.prm, self.cb,
                                  rec=self.rec, count=self.count, ws=self.ws_bin,
                                  out=dict(pair_gid=self.pair_gid,
                                           tile_range=self.tile_range, n_pairs_dev=self.n_pairs),
                                  img=self.img)
        else:
            self.project_bin(view)
            self.forward()

    def check_capacity(self, slots=()):
        """One host read of the status slots (csplat.h) of this view buffer and
        of `slots` (e.g. the window's second view slot): raises if ANY call since
        the last clear overflowed its pair capacity, returns the largest pair
        count seen, and clears the slots."""
        allsl = [self, *[s for s in slots if s is not self]]
        st = torch.stack([cs.range_status(s.tile_range) for s in allsl]).cpu()
        for s in allsl:
            cs.clear_status(s.tile_range)
        bits = int(np.bitwise_or.reduce(st[:, 0].numpy()))
        worst = int(st[:, 1].numpy().view(np.uint32).max())
        cap = min(s.capacity for s in allsl)
        if bits & cs.STATUS_CAPACITY or worst > cap:
            raise cs.CsplatError(f"{worst} pairs exceed the capacity {cap} "
                                 f"(CSPLAT_STATUS_CAPACITY: those tiles were left empty)")
        return worst

    # ---- CUDA graph ------------------------------------------------------
    def capture(self, view, render_only=False):
        """One step (or, render_only, one view's project -> bin -> fwd -> bwd
        incl. the chain, no prune / R-VQ) captured as a CUDA graph."""
        fn = self.render_view if render_only else self.step
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            if render_only:
                self.prepare()
            fn(view)                 # warm (and any lazy attribute setup) outside capture
        torch.cuda.current_stream(self.dev).wait_stream(s)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(view)
        if not render_only:
            self.graph = g
        return g
