import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2403_11247_b200 import csplat as cs, _build
from scenes import synth
_build.build()
dev = torch.device("cuda:0")
sc = synth.mid_scene(4)
g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
H, W = sc.cam["height"], sc.cam["width"]
up = [torch.tensor(a, device=dev) for a in synth.upstream(np.random.default_rng(1), H, W)]
r = cs.render_step(g, sc.cam, sc.views[0], 200000, *up)
obs_c = torch.rand((3, H, W), device=dev); obs_d = torch.rand((H, W), device=dev)
nv = cs.count_valid_depth(obs_d)
out = r[2]; img = r[3]
cs.tracking_step(g, sc.cam, sc.views[0], 200000, obs_c, obs_d, nv, out=out, img=img,
                 rec=torch.empty((g.n, 16), dtype=torch.int32, device=dev),
                 count=torch.empty(g.n, dtype=torch.int32, device=dev))
torch.cuda.synchronize()
print("ok", int(out["n_pairs_dev"].item()))
