"""How many (4x4 block, entry) items the backward's block lists hold at C2 under
the current rule (pixel rectangle inside the pair's 8x8-block mask) and under a
per-pixel test (some pixel of the 4x4 block has q <= k^2): the head-room of a
finer list filter.  `python tools/list_stats.py [c2|c3|c5]` (GPU box)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_11247_b200 import csplat as cs  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from scenes import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda:0")
sc = {"c2": synth.replica_scene, "c3": synth.tum_scene, "c5": synth.window_scene}[cfg](0)
v = sc.views[0]
st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
st.size_pairs(v)
st.prepare()
g = st.pruned
cs.project(g, st.cam, v, st.prm, st.cb, rec=st.rec, count=st.count)
cs.bin_tiles(st.rec, st.count, st.cam, st.capacity, ws=st.ws_bin,
             out=dict(pair_gid=st.pair_gid, tile_range=st.tile_range, n_pairs_dev=st.n_pairs),
             sync=True)
torch.cuda.synchronize()
W, H = sc.cam["width"], sc.cam["height"]
tx_n = (W + 15) // 16
T = tx_n * ((H + 15) // 16)
rec = st.rec.view(torch.float32).reshape(-1, 16).cpu().numpy()
reci = rec.view(np.uint32)
pg = st.pair_gid[: int(st.n_pairs.item())].cpu().numpy().astype(np.uint32)
tr = st.tile_range.view(torch.int32).reshape(-1, 2)[:T].cpu().numpy().view(np.uint32)
tile = np.repeat(np.arange(T), (tr[:, 1] - tr[:, 0]).astype(np.int64))
gid = (pg & 0x0FFFFFFF).astype(np.int64)
m8 = pg >> 28
X0 = (tile % tx_n) * 16
Y0 = (tile // tx_n) * 16
r = rec[gid]
ri = reci[gid]
u, vv, ca, cb2, cc, k2 = r[:, 0], r[:, 1], r[:, 2], r[:, 3], r[:, 4], r[:, 6]
rx0 = (ri[:, 12] & 0xFFFF).astype(np.int64) - X0
ry0 = (ri[:, 12] >> 16).astype(np.int64) - Y0
rx1 = (ri[:, 13] & 0xFFFF).astype(np.int64) - X0
ry1 = (ri[:, 13] >> 16).astype(np.int64) - Y0
cur = 0
fine = 0
pix = 0
for b in range(16):
    qx, qy = b & 3, b >> 2
    inrect = ~((rx1 < 4 * qx) | (rx0 > 4 * qx + 3) | (ry1 < 4 * qy) | (ry0 > 4 * qy + 3))
    in8 = ((m8 >> ((qx >> 1) + 2 * (qy >> 1))) & 1).astype(bool)
    c = inrect & in8
    cur += int(c.sum())
    # per pixel of the block: q <= k^2
    hit = np.zeros(len(pg), bool)
    npx = np.zeros(len(pg), np.int64)
    for yy in range(4):
        for xx in range(4):
            dx = (X0 + 4 * qx + xx) - u
            dy = (Y0 + 4 * qy + yy) - vv
            q = ca * dx * dx + cb2 * dx * dy + cc * dy * dy
            ok = c & (q <= k2)
            hit |= ok
            npx += ok
    fine += int(hit.sum())
    pix += int(npx.sum())
print(f"{cfg}: pairs {len(pg)} tiles {T} (block, entry) items: current {cur} "
      f"per-pixel-exact {fine} ({fine / max(cur, 1):.3f}); (pixel, entry) within k^2: {pix} "
      f"= {pix / max(cur * 16, 1):.3f} of the current items' pixels")
