"""Run a few C2 steps (non-graph launches) for ncu: `python tools/prof_step.py [steps]`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11247_b200 import _build  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from scenes import synth  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    which = sys.argv[2] if len(sys.argv) > 2 else "replica"
    _build.build()
    dev = torch.device("cuda:0")
    sc = synth.replica_scene(0) if which == "replica" else synth.tum_scene(0)
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    v = sc.views[0]
    st.size_pairs(v)
    H, W = sc.cam["height"], sc.cam["width"]
    st.set_upstream(*(torch.tensor(a, device=dev)
                      for a in synth.upstream(np.random.default_rng(1), H, W)))
    for _ in range(steps):
        st.step(v)
    torch.cuda.synchronize()
    print("pairs", int(st.n_pairs.item()), "kept", int(st.n_kept.item()))


if __name__ == "__main__":
    main()
