"""Per-stage device times of one keyframe render (no L2 flush, CUDA events):
python tools/c5_stages.py [keyframe] [c5|c3] -- C5: 64 keyframes x 500k
Gaussians, R-VQ 4x256; C3: TUM 640x480, 100k Gaussians, the tracking pose."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11247_b200 import csplat as cs  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from scenes import synth  # noqa: E402

kf = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
dev = torch.device("cuda:0")
if cfg == "c2":
    sc = synth.replica_scene(0)
    v = sc.views[0]
elif cfg == "c3":
    sc = synth.tum_scene(0)
    v = synth.perturbed_view(np.random.default_rng(11), rot_deg=1.0, trans=0.02)
else:
    sc = synth.window_scene(0)
    v = sc.views[kf]
st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
st.size_pairs(v)
H, W = sc.cam["height"], sc.cam["width"]
st.set_upstream(*(torch.tensor(a, device=dev) for a in synth.upstream(np.random.default_rng(5), H, W)))
st.prepare()
g = st.pruned
stages = [
    ("project", lambda: cs.project(g, st.cam, v, st.prm, st.cb, rec=st.rec, count=st.count)),
    ("bin_tiles", lambda: cs.bin_tiles(st.rec, st.count, st.cam, st.capacity, ws=st.ws_bin,
                                       out=dict(pair_gid=st.pair_gid,
                                                tile_range=st.tile_range, n_pairs_dev=st.n_pairs),
                                       sync=False)),
    ("render_fwd", st.forward),
    ("render_bwd", lambda: st.backward(v, flags=cs.ACCUMULATE)),
]
stream = torch.cuda.current_stream(dev)
acc = {k: [] for k, _ in stages}
t_end = time.time() + 1.5  # soak: clocks up before timing
while time.time() < t_end:
    for _, fn in stages:
        fn()
    torch.cuda.synchronize()
for it in range(22):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * len(stages))]
    for i, (k, fn) in enumerate(stages):
        torch.cuda._sleep(200000)  # keep the GPU busy while the host enqueues the stage
        ev[2 * i].record(stream)
        fn()
        ev[2 * i + 1].record(stream)
    torch.cuda.synchronize()
    if it >= 2:
        for i, (k, _) in enumerate(stages):
            acc[k].append(ev[2 * i].elapsed_time(ev[2 * i + 1]) * 1e3)
print({k: round(statistics.median(x), 1) for k, x in acc.items()},
      "n_kept", int(st.n_kept.item()), "pairs", int(st.n_pairs.item()),
      "in view", int((st.count > 0).sum().item()))
