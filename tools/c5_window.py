"""C5 window iteration on one GPU: the two-slot pipelined window vs the batched
window (multi-view projection + chain), eager and as a CUDA graph.
usage: python tools/c5_window.py [n_keyframes]"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from paper_2403_11247_b200.window import gpu_window  # noqa: E402
from scenes import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda:0")
sc = synth.window_scene(0)
views = sc.views[:K]
st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
st.size_pairs(views[0], views=views[1:])
H, W = sc.cam["height"], sc.cam["width"]
st.set_upstream(*(torch.tensor(a, device=dev) for a in synth.upstream(np.random.default_rng(5), H, W)))
stream = torch.cuda.current_stream(dev)
res = {}
for mode in ("pipelined", "batched", "batched_chainviews"):
    win = gpu_window(st, views, rank=0, world=1, pipelined=True, batched=mode != "pipelined",
                     chain_views=mode == "batched_chainviews")
    win.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        win.run()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        win.run()
    stream.wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        win.run()
    gs = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        gs.append(a.elapsed_time(b))
    flat = st.grads["flat"].clone()
    res[mode] = (statistics.median(ts), statistics.median(gs), flat)
    print(mode, "eager ms", round(res[mode][0], 3), "graph ms", round(res[mode][1], 3), flush=True)
a, b = res["pipelined"][2].double(), res["batched"][2].double()
print("rel diff", float((a - b).norm() / a.norm()))
