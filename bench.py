#!/usr/bin/env python
"""bench.py -- the hot path of arXiv 2403.11247 on B200 (BASELINE.json metric:
"fwd+bwd renders/sec and Gaussian-pixel evals/sec at 1200x680; % HBM/FP32 peak").

One STEP = one pass of every SURVEY.md §8(a) row over one Replica-shaped view
(config C2: 1200x680, 200k Gaussians, 75% mask-kept, R-VQ 4 x 256):
    mask_prune -> rvq_assign (scale, rotation) -> project (mask + R-VQ decode)
    -> bin_tiles -> render_fwd -> render_bwd (chain, STE mask, pose)
captured once as a CUDA graph and replayed.  With --gpus N (torchrun, one rank
per GPU) every rank renders its own keyframe view of the replicated map and the
15-plane gradient buffer is summed with one NCCL all-reduce per step (the
keyframe-window data parallelism of SURVEY.md §8(e)); value = N renders / the
slowest rank's step time (weak scaling).

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the launching stream, with a 512 MB L2-flush write between steps (outside
the events); barrier + synchronize around the timed region; max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fwd+bwd renders/sec at 1200x680 (Replica-shaped, 200k Gaussians)"
UNIT = "renders/s"
def c2_config(world: int) -> dict:
    """The workload both arms report (the GPU step and the oracle reference)."""
    return {"workload": "C2 replica 1200x680, 200k Gaussians (75% kept), R-VQ 4x256, "
                        "step = prune+rvq+project+bin+fwd+bwd"
                        + (" + grad all-reduce" if world > 1 else ""),
            "l2": "512 MB flush write between timed steps",
            "views": "rank r renders its own keyframe (rank 0 identity)",
            "parallelism": f"dp{world} keyframe window"}
KERNEL_LAUNCHES_PER_STEP = {
    # kernels of libcsplat launched by one RenderStep.step(): the projection
    # carries the bucket pass, and the per-tile sort, the forward and the
    # backward kernel run as 2 tile chunks each, then the chain (csplat_render_step)
    "mask_prune": 1, "rvq_assign": 2, "project": 1, "bin_tiles": 2, "render_fwd": 2,
    "render_bwd": 3,
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="csplat", choices=["csplat", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tracking", action="store_true")
    ap.add_argument("--profile-stages", action="store_true", default=True)
    return ap.parse_args()


# ---------------------------------------------------------------- helpers

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, nm in enumerate(names):
                if len(s) > 5 + k and s[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def fp32_peak_tinstr(sm_mhz):
    """FP32 lane-instruction peak: 148 SMs x 128 FP32 lanes x SM clock (B200
    unit counts, /opt/skills/guides/B200_PROFILING.md); FFMA counts as one."""
    return 148 * 128 * sm_mhz * 1e6 / 1e12


def stage_rooflines(stage_ms, counts, n_kept, n_pairs, e_bwd, peaks, step):
    """Algorithmic work per unit x units / measured stage time,
    against the measured HBM copy bandwidth or the FP32 lane-issue peak."""
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    fp = fp32_peak_tinstr(sm_mhz)
    hbm = peaks["hbm_gbs"]
    n = step.n
    L, P = (step.cb.scale_codes.shape[0], step.cb.scale_codes.shape[1]) if step.cb else (0, 0)
    out = {}

    def hb(name, nbytes):
        if name in stage_ms:
            a = nbytes / (stage_ms[name] * 1e-3) / 1e9
            out[name] = {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s",
                         "frac": a / hbm, "bytes": nbytes}

    def al(name, work):
        if name in stage_ms:
            a = work / (stage_ms[name] * 1e-3) / 1e12
            out[name] = {"bound": "alu", "achieved": a, "peak": fp, "unit": "T FP32-lane-op/s",
                         "frac": a / fp, "work": work}

    # SURVEY §8(d) "algorithmic work per unit" (what the method must move / issue);
    # "impl_bytes" = what this implementation moves by design, for comparison
    hb("mask_prune", n * (4 + 60 + 2 * L) + n_kept * (60 + 2 * L))
    if L:
        al("rvq_assign", n_kept * L * P * (2 * 3 + 2 * 4))  # sub + fma per dimension
    hb("project", n_kept * (40 + 60) if L else n_kept * 120)
    if "project" in out:
        out["project"]["impl_bytes"] = 4 * n + n_kept * (32 + 2 * L) + 68 * n
    hb("bin_tiles", 12 * n_kept + (12 + 28) * n_pairs)   # a4 12 B/G + 12 B/pair; a5 28 B/pair
    if "bin_tiles" in out:
        b = 24 * n + 148 * n_pairs  # keys, cursors, pair_gid, 64-B payload gather + write
        out["bin_tiles"]["impl_bytes"] = b
        out["bin_tiles"]["impl_gbs"] = b / (stage_ms["bin_tiles"] * 1e-3) / 1e9
    if counts:
        al("render_fwd", 10.0 * counts["e_pix"] + 11.0 * counts["e_contrib"])
        al("render_bwd_kernel", 10.0 * e_bwd + 35.0 * counts["e_contrib"])
    if "render_bwd" in stage_ms and "render_bwd_kernel" in stage_ms:
        hb("chain", 160 * n_kept)  # a8: 160 B/G
        ch = stage_ms["render_bwd"] - stage_ms["render_bwd_kernel"]
        if ch > 0:
            a = 160 * n_kept / (ch * 1e-3) / 1e9
            out["chain"] = {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s",
                            "frac": a / hbm, "bytes": 160 * n_kept,
                            "ms": ch, "note": "render_bwd - render_bwd_kernel"}
    return out


def bench_tracking(dev, flush, iters=40, frames=3):
    """NEXT-1 on config C3: TUM-shaped 640x480, 100k Gaussians, R-VQ 4x256;
    observed images rendered at the true pose; each frame = 40 pose-only
    iterations (project, bin, fwd, tracking loss, bwd POSE_ONLY, host pose
    step) from a 1 deg / 2 cm perturbation.  CUDA-event timed per frame."""
    import torch
    from paper_2403_11247_b200 import csplat as cs
    from paper_2403_11247_b200.pipeline import RenderStep
    from paper_2403_11247_b200.tracking import Tracker, pose_error
    from scenes import synth
    sc = synth.tum_scene(0)
    gt = sc.views[0]
    start = synth.perturbed_view(np.random.default_rng(11), rot_deg=1.0, trans=0.02)
    obs = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    obs.size_pairs(gt)
    obs.front(gt)
    obs.forward()
    obs_c, obs_d = obs.img["color"].clone(), obs.img["depth"].clone()
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev, flags=cs.POSE_ONLY)
    st.size_pairs(start, views=[gt])
    tr = Tracker(st, obs_c, obs_d)
    tr.track(start, iters=3)  # warm-up
    stream = torch.cuda.current_stream(dev)
    times, errs, losses = [], [], None
    for _ in range(frames):
        flush.fill_(1.0)
        tr.step.prepare()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        view, losses = tr.track(start, iters=iters, lr_rot=5e-4, lr_trans=5e-4)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        errs.append(pose_error(view, gt))
    st.check_capacity()
    ms_host = statistics.median(times)
    # device-resident pose: one iteration captured as a CUDA graph, 40 replays
    tr.capture(start, lr_rot=5e-4, lr_trans=5e-4)
    times, gerrs = [], []
    for _ in range(frames):
        flush.fill_(1.0)
        tr.step.prepare()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        view = tr.track_graph(start, iters=iters)  # ends with the 48-byte view read
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        gerrs.append(pose_error(view, gt))
    st.check_capacity()
    ms = statistics.median(times)
    return {"workload": "C3 TUM 640x480, 100k Gaussians, R-VQ 4x256, pose-only",
            "iters_per_frame": iters, "ms_per_frame": ms, "ms_per_iter": ms / iters,
            "iters_per_s": 1e3 * iters / ms, "frames_per_s": 1e3 / ms,
            "loss_first_last_host_loop": [losses[0], losses[-1]],
            "pose_err_start_deg_m": list(pose_error(start, gt)),
            "pose_err_end_deg_m": list(gerrs[-1]),
            "pose_err_end_deg_m_host_loop": list(errs[-1]),
            "ms_per_iter_host_loop": ms_host / iters,
            "note": "device-resident pose (csplat_pose_step), one iteration captured as a CUDA "
                    "graph and replayed 40x per frame; host_loop = pose step on the host with "
                    "one 36-byte device->host read per iteration"}


def bench_next_rows(step, sc, view, dev, flush, reps=20):
    """Device times of the NEXT-2/3 kernels on the C2 map (CUDA events, cold L2):
    R-VQ codebook update of both attributes over the survivors, the Eq 8 mask
    loss, and keyframe overlap of a 1200x680 depth map against 64 keyframes."""
    import torch
    from paper_2403_11247_b200 import csplat as cs
    from scenes import synth
    stream = torch.cuda.current_stream(dev)
    step.prepare()
    step.project_bin(view)
    step.forward()
    g = step.pruned
    d_mask = torch.zeros(step.n, device=dev)
    win = synth.window_scene(0, n=1000, n_keyframes=64)
    depth = step.img["depth"]
    varr = cs.view_array(win.views)  # marshalled once, outside the timed region
    ov_counts = torch.zeros(len(win.views), dtype=torch.int64, device=dev)
    ov_ws = torch.empty(cs.workspace_bytes(cs.OP_KEYFRAME_OVERLAP, len(win.views)),
                        dtype=torch.uint8, device=dev)
    jobs = {
        "rvq_update_scale_rot": lambda: (cs.rvq_update(g.log_scale, step.cb.scale_codes,
                                                       step.cb.scale_idx, n_dev=step.n_kept),
                                         cs.rvq_update(g.quat, step.cb.rot_codes,
                                                       step.cb.rot_idx, n_dev=step.n_kept)),
        "mask_loss": lambda: cs.mask_loss(g, step.count, d_mask),
        "keyframe_overlap_64": lambda: cs.keyframe_overlap(depth, sc.cam, view, varr,
                                                           counts=ov_counts, ws=ov_ws),
    }
    out = {}
    for name, fn in jobs.items():
        fn()
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        out[name + "_us"] = statistics.median(ts)
    n_kept = int(step.n_kept.item())
    L = step.cb.scale_codes.shape[0]
    out["rvq_update_hbm_gbs"] = n_kept * (4 * 7 + 2 * L) / (out["rvq_update_scale_rot_us"] * 1e-6) / 1e9
    out["keyframe_overlap_points"] = int((depth > 0).sum().item())
    return out


def bench_ba(dev, n_rays=65536, iters=5):
    """NEXT-4: one random-ray global-BA iteration (reading R30) over
    the C5 keyframe database (64 Replica-shaped keyframes x 500k Gaussians,
    R-VQ 4x256): n_rays rays as n_rays/64 random 8x8 patches; per keyframe
    project -> active-tile bin -> fwd -> patch loss (Eq 12 + SSIM) -> bwd
    ACCUMULATE.  Observed images: renders of the map at the keyframe views
    (synthetic).  Device time per iteration (CUDA events, median)."""
    import torch
    from paper_2403_11247_b200 import csplat as cs
    from paper_2403_11247_b200.ba import BatchedBA, ba_loss_value
    from paper_2403_11247_b200.pipeline import RenderStep
    from scenes import synth
    sc = synth.window_scene(0)
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    st.size_pairs(sc.views[0], views=sc.views[1:])
    st.prepare()
    oc, od = [], []
    for v in sc.views:  # observations: the map rendered at the keyframe views
        st.project_bin(v)
        st.forward()
        oc.append(st.img["color"].clone())
        od.append(st.img["depth"].clone())
    patches = synth.sample_patches(1, len(sc.views), sc.cam["width"], sc.cam["height"], n_rays)
    ba = BatchedBA(st, sc.views, oc, od, patches, rank=0, world=1)
    stream = torch.cuda.current_stream(dev)
    ba.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ba.run()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms_eager = statistics.median(ts)
    # the whole iteration (64 keyframes, ~700 launches) captured as one CUDA graph
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        ba.run()
    stream.wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ba.run()
    graph.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        graph.replay()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    max_pairs = ba.check_capacity()  # every keyframe of every timed iteration
    return {"workload": "C5 DB: 64 keyframes x 500k Gaussians, R-VQ 4x256, "
                        f"{ba.n_rays} rays as {ba.n_rays // 64} random 8x8 patches",
            "ms_per_iter": ms, "rays_per_s": ba.n_rays / (ms * 1e-3),
            "n_valid": int(ba.n_valid.item()), "loss": ba_loss_value(ba.loss3),
            "max_pairs_per_kf": max_pairs, "ms_per_iter_eager": ms_eager,
            "note": "graph replay of the whole iteration; eager = per-keyframe host loop"}


def cpu_model() -> str:
    """The host CPU (lscpu 'Model name'), for the oracle baselines."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _timed(fn, stream, flush, reps):
    import torch
    fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def bench_c4(dev, flush, reps=10):
    """C4: ScanNet-shaped 1M unpruned Gaussians: csplat_mask_prune
    over all 1M (keep 1/1.97) and csplat_rvq_assign 4 x 256 of scale and
    rotation over all 1M.  Cold L2, CUDA events, median."""
    import torch
    from paper_2403_11247_b200 import csplat as cs
    from scenes import synth
    sc = synth.scannet_scene(0)
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    n = g.n
    out = cs.GaussianMap(**{k: torch.empty_like(getattr(g, k)) for k in
                            ("mean", "opacity", "rgb", "log_scale", "quat", "mask")})
    keep_map = torch.empty(n, dtype=torch.int32, device=dev)
    n_kept = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(cs.workspace_bytes(cs.OP_MASK_PRUNE, n), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    t_prune = _timed(lambda: cs.mask_prune(g, out=out, keep_map=keep_map, n_kept=n_kept, ws=ws),
                     stream, flush, reps)
    k = int(n_kept.item())
    sct = torch.tensor(sc.codebook["scale_codes"], device=dev)
    rct = torch.tensor(sc.codebook["rot_codes"], device=dev)
    L = sct.shape[0]
    si = torch.empty((L, n), dtype=torch.uint8, device=dev)
    ri = torch.empty((L, n), dtype=torch.uint8, device=dev)
    t_rvq = _timed(lambda: (cs.rvq_assign(g.log_scale, sct, idx=si, want_recon=False),
                            cs.rvq_assign(g.quat, rct, idx=ri, want_recon=False)),
                   stream, flush, reps)
    pbytes = n * (4 + 60) + k * (60 + 4)   # masks + planes read, planes + keep_map written
    work = n * L * sct.shape[1] * (2 * 3 + 2 * 4)  # sub + fma per dimension (stage_rooflines)
    return {"workload": "C4 ScanNet-shaped 1M Gaussians (mask keep 1/1.97), R-VQ 4x256",
            "n": n, "n_kept": k, "prune_us": t_prune,
            "prune_hbm_gbs": pbytes / (t_prune * 1e-6) / 1e9,
            "rvq_scale_rot_us": t_rvq, "rvq_gaussians_per_s": n / (t_rvq * 1e-6),
            "rvq_tlane_ops_per_s": work / (t_rvq * 1e-6) / 1e12}


def bench_c5_window(dev, rank, world, iters=3):
    """C5 (SURVEY §8(d,e)): the mapping window of 64 Replica-shaped keyframes x
    500k Gaussians (R-VQ 4x256) sharded over the ranks (keyframe i -> rank
    i mod G): each rank renders its keyframes fwd+bwd (ACCUMULATE, the local
    part captured as one CUDA graph), then one NCCL all-reduce of the flat
    gradient buffer.  Window iteration time = max over ranks (CUDA events)."""
    import torch
    import torch.distributed as dist
    from paper_2403_11247_b200.pipeline import RenderStep
    from paper_2403_11247_b200.window import gpu_window
    from scenes import synth
    sc = synth.window_scene(0)
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    st.size_pairs(sc.views[rank], views=sc.views[rank + world::world])  # every local keyframe
    H, W = sc.cam["height"], sc.cam["width"]
    st.set_upstream(*(torch.tensor(a, device=dev)
                      for a in synth.upstream(np.random.default_rng(5), H, W)))
    # the local part (the rank's keyframes, multi-view front: one projection
    # read per Gaussian for all of them); the all-reduce is issued below
    win = gpu_window(st, sc.views, rank=rank, world=world, reduce=False, batched=True)
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        win.run()
    stream.wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        win.run()

    def one(ev=None):
        graph.replay()
        if world > 1:
            if ev is not None:
                ev.record(stream)
            dist.all_reduce(st.grads["flat"])

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ts, ars = [], []
    for _ in range(iters):
        a, b, m = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        one(m)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        ars.append(m.elapsed_time(b) if world > 1 else 0.0)
    win.check_capacity()  # every keyframe of every timed iteration, both view slots
    t = statistics.median(ts)
    t_local = t - statistics.median(ars)
    # every rank must hold the identical reduced gradient (the replicas stay in step)
    chk = st.grads["flat"].double().sum().reshape(1)
    same = True
    if world > 1:
        tt = torch.tensor([t], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        lo, hi = chk.clone(), chk.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        same = bool(torch.equal(lo, hi))
        mine = torch.tensor([t_local, statistics.median(ars)], device=dev, dtype=torch.float64)
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per = [tuple(float(x) for x in a_.cpu()) for a_ in allr]
    else:
        per = [(t_local, 0.0)]
    coll = (dist.get_backend().upper() if world > 1 else "NCCL") + " all-reduce"
    return {"workload": "C5 window: 64 keyframes x 500k Gaussians, R-VQ 4x256, "
                        f"keyframes sharded over {world} GPU(s) + {coll}",
            "n_gpus": world, "keyframes_per_rank": len(win.local), "ms_per_window_iter": t,
            "window_iters_per_s": 1e3 / t, "keyframe_renders_per_s": 64e3 / t,
            "reduced_grad_checksum": float(chk.item()), "replicas_identical": same,
            "per_rank_local_ms": [round(p[0], 4) for p in per],
            "per_rank_allreduce_ms": [round(p[1], 4) for p in per],
            "allreduce_share": max(p[1] for p in per) / t,
            "allreduce_bytes": st.grads["flat"].numel() * 4,
            "note": "local part = the rank's keyframes as one CUDA graph; then one SUM "
                    "all-reduce of the flat [15n+8] gradient buffer (time = max over ranks)"}


# ---------------------------------------------------------------- oracle (CPU) legs

def nccl_info(rank: int) -> dict | None:
    """What NCCL chose on this rank (from its INIT/TUNING log): NVLS or not."""
    p = os.path.join(ROOT, "gpurun_out", f"nccl_rank{rank}.log")
    if not os.path.exists(p):
        return None
    txt = open(p, errors="replace").read()
    lines = txt.splitlines()
    pick = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines
            if "NVLS" in ln or "NCCL version" in ln or "comm " in ln and "nRanks" in ln]
    return {"log": os.path.relpath(p, ROOT), "nvls_mentioned": "NVLS" in txt,
            "nvls_enabled": any("NVLS" in ln and ("enabled" in ln.lower() or "support" in
                                                  ln.lower()) for ln in lines),
            "lines": pick[:8]}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _planes_of(outs, k):
    names = ["mean", "opacity", "rgb", "log_scale", "quat", "mask"]
    pl, off = {}, 0
    for name, c in zip(names, (3, 1, 3, 3, 4, 1)):
        pl[name] = np.stack(outs[off:off + c]).reshape((c, k) if c > 1 else (k,))
        off += c
    return pl


def _flat_planes(sc):
    planes = []
    for k in ["mean", "opacity", "rgb", "log_scale", "quat", "mask"]:
        planes += list(getattr(sc, k).reshape(-1, sc.n))
    return planes


def oracle_step(sc, view, upstream, row_frac=1.0):
    """One step of the C2 workload through the CPU oracle as it stands: prune,
    R-VQ (scale + rotation) of every survivor, project, bin, and forward +
    backward (incl. the chain) over the first row_frac of the pixel rows.
    Returns (seconds, render-equivalent seconds, counters): every component
    is timed on its own and charged by the share of one render it covered
    (prune / R-VQ / project / bin / chain: all of it; the per-pixel forward and
    backward: row_frac), so a row-sampled step is not charged a full render's
    prune, projection and binning for a fraction of the pixels."""
    import oracle
    oracle.build()
    H = sc.cam["height"]
    T = {}
    t = time.perf_counter()
    outs, _, _, k = oracle.mask_prune(_flat_planes(sc), [], mask_plane=14)
    pl = _planes_of(outs, k)
    T["prune"] = time.perf_counter() - t
    t = time.perf_counter()
    si, _ = oracle.rvq_assign(pl["log_scale"], sc.codebook["scale_codes"])
    ri, _ = oracle.rvq_assign(pl["quat"], sc.codebook["rot_codes"])
    T["rvq"] = time.perf_counter() - t
    cbo = dict(scale_codes=sc.codebook["scale_codes"], rot_codes=sc.codebook["rot_codes"],
               scale_idx=si, rot_idx=ri)
    S = oracle.Scene(**pl)
    t = time.perf_counter()
    rec, cnt = oracle.project(S, sc.cam, view, codebook=cbo)
    T["project"] = time.perf_counter() - t
    t = time.perf_counter()
    gid, rng = oracle.bin_tiles(rec, cnt, sc.cam)
    T["bin"] = time.perf_counter() - t
    rows = max(1, int(round(H * row_frac)))
    frac = rows / H
    oracle.set_row_window(0, rows)
    try:
        t = time.perf_counter()
        fo = oracle.render_fwd(rec, gid, rng, sc.cam)
        T["fwd"] = time.perf_counter() - t
        dC, dD, dS = upstream
        t = time.perf_counter()
        oracle.render_bwd(S, sc.cam, view, rec, gid, rng, dC, dD, dS, codebook=cbo)
        T["bwd"] = time.perf_counter() - t
    finally:
        oracle.set_row_window(0, -1)
    total = sum(T.values())
    equiv = total - T["fwd"] - T["bwd"] + (T["fwd"] + T["bwd"]) / frac
    return total, equiv, dict(fo=fo, parts=T, row_frac=frac)


def _oracle_render(orc, S, cam, view, up=None, cbo=None):
    rec, cnt = orc.project(S, cam, view, codebook=cbo)
    gid, rng = orc.bin_tiles(rec, cnt, cam)
    fo = orc.render_fwd(rec, gid, rng, cam)
    if up is not None:
        orc.render_bwd(S, cam, view, rec, gid, rng, *up, codebook=cbo)
    return fo


def cpu_configs(threads):
    """SURVEY §8(d) "Oracle timing beside it": the CPU oracle as it stands on
    `threads` host threads, one bounded run per config (extrapolations
    labelled).  Returns {config: {...}}."""
    import oracle
    from scenes import synth
    oracle.build()
    oracle.set_threads(threads)
    out = {}
    try:
        # C1: the whole tiny step (R-VQ 2x16, prune, project, bin, fwd, bwd)
        sc = synth.tiny_scene(0)
        up = synth.upstream(np.random.default_rng(1), sc.cam["height"], sc.cam["width"])
        t = time.perf_counter()
        reps = 20
        for _ in range(reps):
            oracle_step(sc, sc.views[0], up)
        dt = (time.perf_counter() - t) / reps
        out["C1"] = {"ms_per_step": 1e3 * dt, "steps_per_s": 1 / dt, "sample": "20 whole steps"}
        # C2: one whole step (row sampling only if it would take too long)
        sc = synth.replica_scene(0)
        up = synth.upstream(np.random.default_rng(1), sc.cam["height"], sc.cam["width"])
        wall, equiv, info = oracle_step(sc, sc.views[0], up)
        out["C2"] = {"ms_per_render": 1e3 * equiv, "renders_per_s": 1 / equiv,
                     "parts_ms": {k: round(1e3 * v, 1) for k, v in info["parts"].items()},
                     "sample": "1 whole step (prune, R-VQ 2x4x256 of all survivors, project, "
                               "bin, fwd+bwd over all 1200x680 pixels)"}
        # C3: one tracking iteration (project, bin, fwd, Eq 12+14 loss, bwd) x 40
        sc = synth.tum_scene(0)
        keep = sc.mask > oracle.mask_tau(0.01)
        pl = {k: v[..., keep] for k, v in sc.planes().items()}
        si, _ = oracle.rvq_assign(pl["log_scale"], sc.codebook["scale_codes"])
        ri, _ = oracle.rvq_assign(pl["quat"], sc.codebook["rot_codes"])
        cbo = dict(scale_codes=sc.codebook["scale_codes"], rot_codes=sc.codebook["rot_codes"],
                   scale_idx=si, rot_idx=ri)
        S = oracle.Scene(**pl)
        obs = _oracle_render(oracle, S, sc.cam, sc.views[0], cbo=cbo)
        start = synth.perturbed_view(np.random.default_rng(11), rot_deg=1.0, trans=0.02)
        t = time.perf_counter()
        rec, cnt = oracle.project(S, sc.cam, start, codebook=cbo)
        gid, rng = oracle.bin_tiles(rec, cnt, sc.cam)
        fo = oracle.render_fwd(rec, gid, rng, sc.cam)
        up, _, _ = oracle.tracking_loss(fo["color"], fo["depth"], fo["sil"], obs["color"],
                                        obs["depth"])
        oracle.render_bwd(S, sc.cam, start, rec, gid, rng, *up, codebook=cbo)
        dt = time.perf_counter() - t
        out["C3"] = {"ms_per_iter": 1e3 * dt, "ms_per_frame_extrapolated": 40e3 * dt,
                     "sample": "1 tracking iteration; per frame = x40 (extrapolation)"}
        # C4: prune over all 1M + R-VQ 4x256 (scale, rotation) over 1/16 of them x 16
        sc = synth.scannet_scene(0)
        t = time.perf_counter()
        oracle.mask_prune(_flat_planes(sc), [], mask_plane=14)
        t_prune = time.perf_counter() - t
        m = sc.n // 16
        t = time.perf_counter()
        oracle.rvq_assign(np.ascontiguousarray(sc.log_scale[:, :m]), sc.codebook["scale_codes"])
        oracle.rvq_assign(np.ascontiguousarray(sc.quat[:, :m]), sc.codebook["rot_codes"])
        t_rvq = (time.perf_counter() - t) * sc.n / m
        out["C4"] = {"prune_ms": 1e3 * t_prune, "rvq_ms_extrapolated": 1e3 * t_rvq,
                     "sample": f"prune of all {sc.n}; R-VQ of the first {m} (1/16), x16"}
        # C5: one keyframe fwd+bwd of the 500k map; a window = 64/G keyframes
        sc = synth.window_scene(0)
        keep = sc.mask > oracle.mask_tau(0.01)
        pl = {k: v[..., keep] for k, v in sc.planes().items()}
        si, _ = oracle.rvq_assign(pl["log_scale"], sc.codebook["scale_codes"])
        ri, _ = oracle.rvq_assign(pl["quat"], sc.codebook["rot_codes"])
        cbo = dict(scale_codes=sc.codebook["scale_codes"], rot_codes=sc.codebook["rot_codes"],
                   scale_idx=si, rot_idx=ri)
        S = oracle.Scene(**pl)
        up = synth.upstream(np.random.default_rng(5), sc.cam["height"], sc.cam["width"])
        t = time.perf_counter()
        _oracle_render(oracle, S, sc.cam, sc.views[0], up=up, cbo=cbo)
        dt = time.perf_counter() - t
        out["C5"] = {"ms_per_keyframe": 1e3 * dt,
                     "ms_per_window_iter_extrapolated_G1": 64e3 * dt,
                     "sample": "1 keyframe fwd+bwd (project, bin, fwd, bwd with chain); "
                               "window = x64/G keyframes (extrapolation, no all-reduce)"}
    finally:
        oracle.set_threads(1)
    return out


def oracle_counts(sc, view):
    """E_pix / E_contrib of the exact scene, counted by the oracle (§8(d))."""
    import oracle
    oracle.build()
    oracle.set_threads(host_cores())
    try:
        keep = sc.mask > oracle.mask_tau(0.01)
        pl = {k: v[..., keep] for k, v in sc.planes().items()}
        si, _ = oracle.rvq_assign(pl["log_scale"], sc.codebook["scale_codes"])
        ri, _ = oracle.rvq_assign(pl["quat"], sc.codebook["rot_codes"])
        cbo = dict(scale_codes=sc.codebook["scale_codes"], rot_codes=sc.codebook["rot_codes"],
                   scale_idx=si, rot_idx=ri)
        rec, cnt = oracle.project(oracle.Scene(**pl), sc.cam, view, codebook=cbo)
        gid, rng = oracle.bin_tiles(rec, cnt, sc.cam)
        fo = oracle.render_fwd(rec, gid, rng, sc.cam)
    finally:
        oracle.set_threads(1)
    return dict(e_pix=fo["e_pix"], e_contrib=fo["e_contrib"], n_pairs=len(gid),
                n_active=int((cnt > 0).sum()), n_kept=int(keep.sum()))


def gpu_local_cpus(dev):
    """The host cores on the GPU's NUMA node (sysfs local_cpulist of its PCI
    device), or an empty set when the platform does not say."""
    import torch
    try:
        pr = torch.cuda.get_device_properties(dev)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        txt = open(f"/sys/bus/pci/devices/{bdf}/local_cpulist").read().strip()
        cpus = set()
        for part in txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        return cpus & os.sched_getaffinity(0)
    except (OSError, ValueError, AttributeError):
        return set()


def cpu_baseline_block():
    """cpu_baseline of the GPU arm: the oracle on 1 thread and on all host cores."""
    n = host_cores()
    one = cpu_configs(1)
    alln = cpu_configs(n) if n > 1 else one
    return {"value": alln["C2"]["renders_per_s"], "unit": UNIT, "cores": n, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": alln["C2"]["sample"] + f", OpenMP {n} threads",
            "single_thread": {"value": one["C2"]["renders_per_s"], "cores": 1},
            "configs": {"threads_1": one, f"threads_{n}": alln}}


def run_reference(args, rank, world):
    """--impl reference: the oracle, as it stands, on all the host's cores, on
    this arm's config / metric / unit.  A step is one C2 render; if whole steps
    would not fit a few minutes, each step renders a band of pixel rows and is
    charged per component (oracle_step)."""
    import oracle
    from scenes import synth
    if rank != 0:
        return
    n = host_cores()
    oracle.build()
    oracle.set_threads(n)
    sc = synth.replica_scene(args.seed)
    view = sc.views[0]
    H, W = sc.cam["height"], sc.cam["width"]
    up = synth.upstream(np.random.default_rng(args.seed + 1), H, W)
    wall0, eq0, _ = oracle_step(sc, view, up)
    budget = 150.0
    frac = 1.0
    if (args.steps + args.warmup) * wall0 > budget:
        frac = max(1.0 / 64, budget / ((args.steps + args.warmup) * wall0))
    walls, eqs = [], []
    for i in range(args.warmup + args.steps):
        w, e, _ = oracle_step(sc, view, up, row_frac=frac)
        if i >= args.warmup:
            walls.append(w)
            eqs.append(e)
    oracle.set_threads(1)
    value = len(eqs) / sum(eqs)
    sample = ("whole C2 steps" if frac == 1.0 else
              f"each step: prune, R-VQ, project, bin over the whole map and fwd+bwd over "
              f"{frac:.3f} of the pixel rows, charged per component")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.mean(walls), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": c2_config(world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": n, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg

def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    from paper_2403_11247_b200 import _build
    from paper_2403_11247_b200 import csplat as cs
    from paper_2403_11247_b200.pipeline import RenderStep
    from scenes import synth

    # one process per GPU; (local % device count) and CSPLAT_DIST_BACKEND=gloo only
    # serve the single-GPU smoke test of the multi-rank code path
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = None
    if world > 1:
        backend = os.environ.get("CSPLAT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # communicator setup per rank (NVLS / channels / algorithms) into
            # gpurun_out/nccl_rank<r>.log; INIT + TUNING only (no per-op logging)
            if os.environ.get("CSPLAT_NCCL_LOG", "1") == "1":
                os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,TUNING,NVLS")
                os.environ.setdefault("NCCL_DEBUG_FILE",
                                      os.path.join(ROOT, "gpurun_out", f"nccl_rank{rank}.log"))
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        if local == 0:
            _build.build()       # one rank (re)builds the in-tree library, the others wait
        dist.barrier()
    else:
        _build.build()
    sc = synth.replica_scene(args.seed)
    H, W = sc.cam["height"], sc.cam["width"]
    # keyframe view of this rank: identity for rank 0, a nearby pose otherwise
    view = sc.views[0] if rank == 0 else synth.perturbed_view(
        np.random.default_rng(1000 + rank), rot_deg=2.0, trans=0.05)
    step = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    step.size_pairs(view)
    up = synth.upstream(np.random.default_rng(args.seed + 1), H, W)
    step.set_upstream(*(torch.tensor(a, device=dev) for a in up))
    graph = step.capture(view)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def one(timed_events=None):
        if timed_events is not None:
            timed_events[0].record(stream)
        graph.replay()
        if world > 1:
            if timed_events is not None:
                timed_events[2].record(stream)
            dist.all_reduce(step.grads["flat"])
        if timed_events is not None:
            timed_events[1].record(stream)

    clocks = ClockSampler(local)
    with clocks:
        for _ in range(args.warmup):
            one()
            flush.fill_(1.0)
        # untimed soak so the clock samples see the GPU under load
        t_end = time.time() + 1.0
        while time.time() < t_end:
            one()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))
               for _ in range(args.steps)]
        for e in evs:
            flush.fill_(1.0)
            one(e)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    step.check_capacity()
    ms = [e[0].elapsed_time(e[1]) for e in evs]
    ar_ms = [e[2].elapsed_time(e[1]) for e in evs] if world > 1 else [0.0] * len(evs)
    t_rank = sum(ms) / 1e3
    if world > 1:
        t = torch.tensor([t_rank], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    else:
        t_max = t_rank
    value = world * args.steps / t_max
    multi = None
    if world > 1:
        # per-rank step time and all-reduce time (device events), gathered to rank 0
        mine = torch.tensor([t_rank * 1e3 / args.steps, statistics.median(ar_ms)],
                            device=dev, dtype=torch.float64)
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per = [tuple(float(x) for x in a.cpu()) for a in allr]
        flat_bytes = step.grads["flat"].numel() * step.grads["flat"].element_size()
        multi = {"backend": backend, "world": world,
                 "per_rank_step_ms": [round(p[0], 4) for p in per],
                 "allreduce_ms_median_per_rank": [round(p[1], 4) for p in per],
                 "allreduce_share": max(p[1] for p in per) / max(p[0] for p in per),
                 "allreduce_bytes": flat_bytes,
                 "allreduce_busbw_gbs": 2 * (world - 1) / world * flat_bytes /
                 (max(p[1] for p in per) * 1e-3) / 1e9 if max(p[1] for p in per) > 0 else None,
                 "nccl": nccl_info(rank) if backend == "nccl" else None}

    # ---- per-stage device times (same stream, non-graph launches, flushed L2)
    stage_ms = {}
    if args.profile_stages:
        g = step.pruned
        stages = [
            ("mask_prune", step.prune),
            ("rvq_assign", step.assign_codes),
            ("project", lambda: cs.project(g, step.cam, view, step.prm, step.cb, rec=step.rec,
                                           count=step.count)),
            ("bin_tiles", lambda: cs.bin_tiles(step.rec, step.count, step.cam, step.capacity,
                                               ws=step.ws_bin,
                                               out=dict(pair_gid=step.pair_gid,
                                                        
                                                        tile_range=step.tile_range,
                                                        n_pairs_dev=step.n_pairs),
                                               sync=False)),
            ("render_fwd", step.forward),
            ("render_bwd", lambda: step.backward(view)),
            # the compositing backward kernel alone (k_render_bwd_quad,
            # CSPLAT_SKIP_CHAIN; its workspace zeroed before the flush, outside
            # the timed region, CSPLAT_WS_ZEROED): the dominant kernel the
            # roofline line reports
            ("render_bwd_kernel", lambda: step.backward(view, flags=cs.SKIP_CHAIN | cs.WS_ZEROED)),
        ]
        pre = {"render_bwd_kernel": lambda: step.ws_bwd.zero_()}
        acc = {k: [] for k, _ in stages}
        for _ in range(max(5, min(args.steps, 30))):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * len(stages))]
            for i, (k, fn) in enumerate(stages):
                if k in pre:
                    pre[k]()
                flush.fill_(1.0)          # every stage starts with a cold L2
                ev[2 * i].record(stream)
                fn()
                ev[2 * i + 1].record(stream)
            torch.cuda.synchronize()
            for i, (k, _) in enumerate(stages):
                acc[k].append(ev[2 * i].elapsed_time(ev[2 * i + 1]))
        stage_ms = {k: statistics.mean(v) for k, v in acc.items()}

    # ---- SURVEY §8(d) metric: one view's project -> bin -> fwd -> bwd (incl. the
    # chain), no prune / R-VQ, captured as a CUDA graph: 20 warm-up + 200 timed
    # replays, median with p10 / p90; warm L2 (no flush, as §8(d) states) and,
    # separately, with the 512 MB flush before each replay
    render_only = None
    if rank == 0:
        g_r = step.capture(view, render_only=True)
        for _ in range(20):
            g_r.replay()
        torch.cuda.synchronize()

        def replays(flush_each):
            out = []
            for _ in range(200):
                if flush_each:
                    flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g_r.replay()
                b.record(stream)
                out.append((a, b))
            torch.cuda.synchronize()
            return sorted(x.elapsed_time(y) for x, y in out)

        warm, cold = replays(False), replays(True)
        q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))]
        render_only = {"renders_per_s": 1e3 / q(warm, 0.5), "ms_median": q(warm, 0.5),
                       "ms_p10": q(warm, 0.1), "ms_p90": q(warm, 0.9),
                       "cold_l2_ms_median": q(cold, 0.5),
                       "cold_l2_renders_per_s": 1e3 / q(cold, 0.5),
                       "note": "csplat_render_step (project+bucket, per-tile sort, fwd, bwd, "
                               "chain) as one CUDA graph, 200 replays; warm L2 unless 'cold'"}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # the pinned staging lives on the GPU's NUMA node: this thread runs on
        # the GPU-local cores while the buffers are allocated and first touched
        # (and while the loop enqueues), so the DMA does not cross sockets
        aff_saved = os.sched_getaffinity(0)
        local = gpu_local_cpus(dev)
        if local:
            os.sched_setaffinity(0, local)
        ins = {k: torch.tensor(v).pin_memory() for k, v in sc.planes().items()}
        up_h = [torch.tensor(a).pin_memory() for a in up]
        outs_h = {k: torch.empty(step.img[k].shape, dtype=step.img[k].dtype).pin_memory()
                  for k in ("color", "depth", "sil")}
        grad_h = torch.empty(step.grads["flat"].shape).pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in ins.values()) + \
            sum(t.numel() * t.element_size() for t in up_h)
        d2h = sum(t.numel() * t.element_size() for t in outs_h.values()) + \
            grad_h.numel() * grad_h.element_size()
        # Pipelined like a streaming user: each step's inputs go host -> device
        # as ONE contiguous copy into a double-buffered staging area on a
        # copy-in stream, the results device -> host as one copy on a copy-out
        # stream (PCIe is full duplex), while the GPU computes the neighbouring
        # step.  On the compute stream a step is the L2 flush and two graph
        # replays: (staging -> the step's buffers, the whole step) and (results
        # -> staging), so the host enqueues ~15 calls per step and stays ahead
        # of the GPU (one copy per tensor was ~50 calls: host-bound at ~0.9 ms).
        # The timed region is the whole K-step loop (CUDA events, streams joined).
        in_src = [ins[k] for k in ins] + up_h
        in_dst = [getattr(step.g, k) for k in ins] + list(step.upstream)
        in_n = [t.numel() for t in in_src]
        in_h = torch.cat([t.reshape(-1) for t in in_src]).pin_memory()
        out_src = [step.img[k] for k in outs_h] + [step.grads["flat"]]
        out_n = [t.numel() for t in out_src]
        st_in = [torch.empty(sum(in_n), device=dev) for _ in range(2)]
        st_out = [torch.empty(sum(out_n), device=dev) for _ in range(2)]
        out_hb = [torch.empty(sum(out_n)).pin_memory() for _ in range(2)]

        def copy_in(buf):
            o = 0
            for dst, m in zip(in_dst, in_n):
                dst.view(-1).copy_(buf[o:o + m])
                o += m

        def copy_out(buf):
            o = 0
            for src, m in zip(out_src, out_n):
                buf[o:o + m].copy_(src.view(-1))
                o += m

        gA, gB = [], []
        for bi in range(2):
            side = torch.cuda.Stream(dev)
            side.wait_stream(stream)
            with torch.cuda.stream(side):  # warm outside capture
                copy_in(st_in[bi])
                step.step(view)
                copy_out(st_out[bi])
            stream.wait_stream(side)
            torch.cuda.synchronize()
            ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(ga):
                copy_in(st_in[bi])
                step.step(view)
            with torch.cuda.graph(gb):
                copy_out(st_out[bi])
            gA.append(ga)
            gB.append(gb)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        in_ready = [torch.cuda.Event() for _ in range(2)]
        in_free = [torch.cuda.Event() for _ in range(2)]
        out_ready = [torch.cuda.Event() for _ in range(2)]
        out_free = [torch.cuda.Event() for _ in range(2)]

        def h2d_issue(j):  # stage step j's inputs in st_in[j % 2]
            bi = j % 2
            with torch.cuda.stream(s_in):
                s_in.wait_event(in_free[bi])
                st_in[bi].copy_(in_h, non_blocking=True)
                in_ready[bi].record(s_in)

        def run(n):
            h2d_issue(0)
            for i in range(n):
                bi = i % 2
                if i + 1 < n:
                    h2d_issue(i + 1)  # the next step's inputs, overlapping this step
                flush.fill_(1.0)
                stream.wait_event(in_ready[bi])
                gA[bi].replay()
                in_free[bi].record(stream)
                if world > 1:
                    dist.all_reduce(step.grads["flat"])
                stream.wait_event(out_free[bi])
                gB[bi].replay()
                out_ready[bi].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(out_ready[bi])
                    out_hb[bi].copy_(st_out[bi], non_blocking=True)
                    out_free[bi].record(s_out)
            stream.wait_stream(s_out)
            stream.wait_stream(s_in)

        for bi in range(2):
            in_free[bi].record(stream)
            out_free[bi].record(stream)
        run(args.warmup)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run(args.steps)
        b.record(stream)
        torch.cuda.synchronize()
        t_e = a.elapsed_time(b) / 1e3
        if world > 1:
            t = torch.tensor([t_e], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e = float(t.item())
        # the host copy of the last step's results equals the device results
        # (images and the flat gradient buffer, bit for bit)
        last = out_hb[(args.steps - 1) % 2]
        ref = torch.cat([t.reshape(-1) for t in out_src]).cpu()
        host_ok = bool(torch.equal(last, ref))
        if local:
            os.sched_setaffinity(0, aff_saved)
        e2e = {"value": world * args.steps / t_e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "host_results_match_device": host_ok,
               "host_cpus": f"{len(local)} GPU-local cores" if local else "no NUMA info",
               "note": "pinned host buffers, one H2D and one D2H copy per step (double-buffered "
                       "device staging); H2D of step i+1 and D2H of step i-1 overlap step i "
                       "(copy streams), whole K-step loop timed on the device, L2 flush inside"}

    # ---- NEXT-1: C3 TUM tracking (40 pose-only iterations per frame), rank 0 only
    tracking = None
    if rank == 0 and not args.no_tracking:
        tracking = bench_tracking(dev, flush)
    next_rows = None
    if rank == 0 and not args.no_tracking:
        next_rows = bench_next_rows(step, sc, view, dev, flush)
        next_rows["global_ba"] = bench_ba(dev)
    c4 = bench_c4(dev, flush) if rank == 0 and not args.no_tracking else None
    # every rank takes part in the sharded C5 window (its collective is a real exchange)
    c5 = None if args.no_tracking else bench_c5_window(dev, rank, world)

    if rank == 0:
        n_kept = int(step.n_kept.item())
        n_pairs = int(step.n_pairs.item())
        e_bwd = int(step.img["n_contrib"].sum().item())
        peaks, peak_src = measured_peaks()
        ck = clocks.summary()
        counts = None
        cpu = None
        if not args.no_cpu_baseline:
            counts = oracle_counts(sc, view)
            cpu = cpu_baseline_block()
        # roofline of the dominant kernel (k_render_bwd: the largest share of the
        # step's kernel time in the ncu launch list, profiles/)
        roof = None
        if stage_ms and counts is not None and "render_bwd_kernel" in stage_ms:
            sm_mhz = peaks.get("sm_max_mhz", 1965.0)
            # §8(d): ~10 lane-instr per replayed entry (E_bwd = sum n_contrib)
            # + ~35 per contributing entry (E_contrib, counted by the oracle)
            work = 10.0 * e_bwd + 35.0 * counts["e_contrib"]
            t_k = stage_ms["render_bwd_kernel"]
            ach = work / (t_k * 1e-3) / 1e12
            peak = fp32_peak_tinstr(sm_mhz)
            roof = {"bound": "alu", "kernel": "k_render_bwd", "achieved": ach, "peak": peak,
                    "unit": "T FP32-lane-instr/s", "frac": ach / peak, "traffic": None,
                    "work_per_launch": work, "ms_per_launch": t_k,
                    "peak_source": f"148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz "
                                   f"(sm_max_mhz of {peak_src} MEASURED_PEAKS.json; "
                                   f"DESIGN.md §8)"}
            tr = os.path.join(ROOT, "profiles", "traffic.json")
            if os.path.exists(tr):
                roof["traffic"] = json.load(open(tr)).get("render_bwd")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": c2_config(world),
            "gpu_launches": sum(KERNEL_LAUNCHES_PER_STEP.values()) * args.steps,
            "stage_ms": stage_ms,
            "n_kept": n_kept, "n_pairs": n_pairs, "e_bwd": e_bwd,
            "clocks": ck,
        }
        if counts:
            line["evals"] = {"e_pix": counts["e_pix"], "e_contrib": counts["e_contrib"],
                             "fwd_evals_per_s": counts["e_pix"] / (stage_ms.get("render_fwd", 0) * 1e-3)
                             if stage_ms.get("render_fwd") else None,
                             "bwd_evals_per_s": e_bwd / (stage_ms.get("render_bwd", 0) * 1e-3)
                             if stage_ms.get("render_bwd") else None}
        if stage_ms:
            # one view's render (project + bin + fwd + bwd) without the per-iteration
            # map maintenance (prune, R-VQ), from the cold-L2 stage times
            line["render_only_fwd_bwd_per_s"] = 1e3 / (stage_ms["project"] + stage_ms["bin_tiles"]
                                                        + stage_ms["render_fwd"]
                                                        + stage_ms["render_bwd"])
            line["stage_roofline"] = stage_rooflines(stage_ms, counts, n_kept, n_pairs, e_bwd,
                                                     peaks, step)
        if c4:
            line["c4_prune_rvq"] = c4
        if c5:
            line["c5_window"] = c5
        if tracking:
            line["tracking_c3"] = tracking
        if next_rows:
            line["next_rows"] = next_rows
        if roof:
            line["roofline"] = roof
        if cpu:
            line["cpu_baseline"] = cpu
        if e2e:
            line["e2e"] = e2e
        if multi:
            line["multi_gpu"] = multi
        if render_only:
            line["render_only_graph"] = render_only
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()           # the other ranks wait for rank 0's CPU-side legs
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
