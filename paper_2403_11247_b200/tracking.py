"""NEXT-1: camera tracking iterations (Sec 3.4) on the csplat path.

One iteration = project -> bin_tiles -> render_fwd -> tracking_loss (Eq 12 gated
by Eq 14) -> render_bwd(POSE_ONLY) -> a fixed-step descent on the left
perturbation xi = (omega, v) of the world->camera pose (R22).  Every stage is a
libcsplat kernel.  Two drivers:

* ``track``: the pose update on the host (one 36-byte device->host read per
  iteration, the view passed to the ABI by value);
* ``track_graph``: the view lives in device memory (``csplat_project_dv`` /
  ``csplat_tracking_bwd`` read it when they run, ``csplat_pose_step`` updates
  it) and the loss is fused into the backward (``csplat_tracking_bwd``: the
  Eq 12 + Eq 14 upstream formed in its prologue, gated-out pixels skipped), so
  one iteration is captured once as a CUDA graph and a frame's iterations are
  graph replays with no host round trip.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import csplat as cs
from .pipeline import FUSED_BIN, RenderStep


def rodrigues(w):
    th = float(np.linalg.norm(w))
    K = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]], dtype=np.float64)
    if th < 1e-12:
        return np.eye(3) + K
    return np.eye(3) + math.sin(th) / th * K + (1 - math.cos(th)) / th ** 2 * (K @ K)


def apply_left(view, xi):
    """V' = Exp(xi) V with p' = Rod(omega) p + v (the perturbation the pose
    gradient of csplat_render_bwd is taken with)."""
    V = np.asarray(view, dtype=np.float64).reshape(3, 4)
    R = rodrigues(np.asarray(xi[:3], dtype=np.float64))
    out = np.empty((3, 4))
    out[:, :3] = R @ V[:, :3]
    out[:, 3] = R @ V[:, 3] + np.asarray(xi[3:], dtype=np.float64)
    return out.astype(np.float32)


def pose_error(view_a, view_b):
    """(rotation angle in degrees, translation distance) between two poses."""
    A = np.asarray(view_a, dtype=np.float64).reshape(3, 4)
    B = np.asarray(view_b, dtype=np.float64).reshape(3, 4)
    Rr = A[:, :3] @ B[:, :3].T
    ang = math.degrees(math.acos(max(-1.0, min(1.0, (np.trace(Rr) - 1) / 2))))
    ca, cb = -A[:, :3].T @ A[:, 3], -B[:, :3].T @ B[:, 3]
    return ang, float(np.linalg.norm(ca - cb))


class Tracker:
    """Pose-only tracking of one frame against observed colour/depth images."""

    def __init__(self, step: RenderStep, obs_color, obs_depth, lambda_depth=1.0,
                 sil_gate=0.99):
        self.step = step
        self.obs_color, self.obs_depth = obs_color, obs_depth
        self.lambda_depth, self.sil_gate = lambda_depth, sil_gate
        dev = step.dev
        self.up = (torch.empty_like(step.img["color"]), torch.empty_like(step.img["depth"]),
                   torch.empty_like(step.img["sil"]))
        self.loss3 = torch.zeros(3, device=dev)
        self.pose = torch.zeros(6, device=dev)
        self.ws = torch.empty(cs.workspace_bytes(cs.OP_TRACKING_LOSS, 0), dtype=torch.uint8,
                              device=dev)
        self.host = torch.empty(9, pin_memory=True)
        self.n_valid = cs.count_valid_depth(obs_depth)  # |R| of the frame (Eq 12), once
        self.step.prepare()   # mask prune + R-VQ of the (fixed) map, once per frame

    def iteration_device(self, view):
        """Enqueue one iteration's kernels (no host synchronisation)."""
        st = self.step
        st.project_bin(view)
        st.forward()
        cs.tracking_loss(st.img, self.obs_color, self.obs_depth, self.lambda_depth,
                         self.sil_gate, out=self.up, loss3=self.loss3, ws=self.ws)
        st.set_upstream(*self.up)
        st.backward(view, flags=cs.POSE_ONLY, pose=self.pose)

    def iteration(self, view, lr_rot, lr_trans):
        self.iteration_device(view)
        self.host[:6].copy_(self.pose, non_blocking=True)
        self.host[6:].copy_(self.loss3, non_blocking=True)
        torch.cuda.current_stream(self.step.dev).synchronize()
        g = self.host.numpy().astype(np.float64)
        xi = np.concatenate([-lr_rot * g[:3], -lr_trans * g[3:6]])
        return apply_left(view, xi), float(g[6])

    def track(self, view, iters=40, lr_rot=1e-4, lr_trans=1e-4):
        losses = []
        for _ in range(iters):
            view, loss = self.iteration(view, lr_rot, lr_trans)
            losses.append(loss)
        return view, losses

    # ---- device-resident pose: a frame's iterations as CUDA-graph replays
    def iteration_dv(self, view_dev, lr_rot, lr_trans):
        """One iteration with the view in device memory (capturable): project ->
        bin -> fwd -> loss-fused backward (Eq 12 + Eq 14 formed in the backward's
        prologue, gated-out pixels not replayed) -> device pose step."""
        st = self.step
        g = st.pruned
        if FUSED_BIN:  # project + bin + fwd + loss-fused bwd per tile chunk, one call
            cs.tracking_step(g, st.cam, view_dev, st.capacity, self.obs_color, self.obs_depth,
                             self.n_valid, st.prm, st.cb, flags=cs.POSE_ONLY,
                             lambda_depth=self.lambda_depth, sil_gate=self.sil_gate,
                             rec=st.rec, count=st.count, ws=st.ws_bin,
                             out=dict(pair_gid=st.pair_gid,
                                      tile_range=st.tile_range, n_pairs_dev=st.n_pairs),
                             img=st.img, grads=dict(st.grads, pose=self.pose),
                             loss3=self.loss3, ws_bwd=st.ws_bwd)
        else:
            st.project_bin_forward(view_dev)
            cs.tracking_bwd(g, st.cam, view_dev, st.rec, st.pair_gid, st.tile_range, st.img,
                            self.obs_color, self.obs_depth, self.n_valid, st.prm, st.cb,
                            flags=cs.POSE_ONLY, lambda_depth=self.lambda_depth,
                            sil_gate=self.sil_gate, grads=dict(st.grads, pose=self.pose),
                            loss3=self.loss3, ws=st.ws_bwd)
        cs.pose_step(view_dev, self.pose, lr_rot, lr_trans)

    def capture(self, view, lr_rot=1e-4, lr_trans=1e-4):
        """Capture one device-pose iteration as a CUDA graph (the pair buffers
        must already be sized: RenderStep.size_pairs)."""
        dev = self.step.dev
        self.view_dev = torch.as_tensor(np.asarray(view, dtype=np.float32).reshape(12)).to(dev)
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):  # warm-up outside the capture
            self.iteration_dv(self.view_dev.clone(), lr_rot, lr_trans)
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.iteration_dv(self.view_dev, lr_rot, lr_trans)
        return self.graph

    def track_graph(self, view, iters=40):
        """A frame's `iters` iterations as graph replays; returns the final view."""
        self.view_dev.copy_(torch.as_tensor(np.asarray(view, dtype=np.float32).reshape(12)))
        for _ in range(iters):
            self.graph.replay()
        return self.view_dev.view(3, 4).cpu().numpy()

