"""How much of k_sort_tiles' latency-bound time can hide under the forward's
compute: time bin (bucket + sort) of view A, forward of view B, back to back
and concurrently on two streams (independent data), CUDA events, C2 scene."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11247_b200 import csplat as cs  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from scenes import synth  # noqa: E402

dev = torch.device("cuda:0")
sc = synth.replica_scene(0)
vA, vB = sc.views[0], synth.perturbed_view(np.random.default_rng(3), rot_deg=2.0, trans=0.05)
A = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
B = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
for st, v in ((A, vA), (B, vB)):
    st.size_pairs(v)
    st.prepare()
    st.project_bin(v)
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
main = torch.cuda.current_stream(dev)


def bin_a():
    cs.bin_tiles(A.rec, A.count, A.cam, A.capacity, ws=A.ws_bin,
                 out=dict(pair_gid=A.pair_gid, tile_range=A.tile_range,
                          n_pairs_dev=A.n_pairs), sync=False)


res = {"serial": [], "concurrent": [], "bin": [], "fwd": []}
for it in range(25):
    for mode in res:
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        if mode == "serial":
            bin_a()
            B.forward()
        elif mode == "bin":
            bin_a()
        elif mode == "fwd":
            B.forward()
        else:
            s1.wait_stream(main)
            s2.wait_stream(main)
            with torch.cuda.stream(s1):
                bin_a()
            with torch.cuda.stream(s2):
                B.forward()
            main.wait_stream(s1)
            main.wait_stream(s2)
        e1.record(main)
        torch.cuda.synchronize()
        if it >= 5:
            res[mode].append(e0.elapsed_time(e1) * 1e3)
print({k: round(statistics.median(v), 1) for k, v in res.items()})
