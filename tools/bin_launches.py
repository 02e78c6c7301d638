"""Run the stand-alone C2 binning (csplat_bin_tiles) a few times for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_11247_b200 import csplat as cs  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from scenes import synth  # noqa: E402

dev = torch.device("cuda:0")
sc = synth.replica_scene(0)
st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
v = sc.views[0]
st.size_pairs(v)
st.prepare()
cs.project(st.pruned, st.cam, v, st.prm, st.cb, rec=st.rec, count=st.count)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    cs.bin_tiles(st.rec, st.count, st.cam, st.capacity, ws=st.ws_bin,
                 out=dict(pair_gid=st.pair_gid, tile_range=st.tile_range, n_pairs_dev=st.n_pairs))
torch.cuda.synchronize()
print("pairs", int(st.n_pairs.item()))
