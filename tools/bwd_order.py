"""Experiment: the C2 backward kernel (CSPLAT_SKIP_CHAIN) in natural tile order vs
list mode with the tiles ordered by list length (heaviest first)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_11247_b200 import csplat as cs  # noqa: E402
from paper_2403_11247_b200.pipeline import RenderStep  # noqa: E402
from scenes import synth  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    sc = synth.replica_scene(0)
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    v = sc.views[0]
    st.size_pairs(v)
    H, W = sc.cam["height"], sc.cam["width"]
    st.set_upstream(*(torch.tensor(a, device=dev) for a in synth.upstream(np.random.default_rng(1), H, W)))
    st.step(v)
    st.project_bin_forward(v)
    torch.cuda.synchronize()
    T = st.tile_range.shape[0] - 1 if st.tile_range.dim() == 2 else st.tile_range.numel() // 2 - 1
    rng = st.tile_range.view(-1, 2)[:T].long()
    ln = (rng[:, 1] - rng[:, 0])
    orders = {"natural": torch.arange(T, device=dev),
              "heavy_first": torch.argsort(ln, descending=True),
              "light_first": torch.argsort(ln)}
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
    dC, dD, dS = st.upstream

    def run(lst):
        if lst is None:
            st.backward(v, flags=cs.SKIP_CHAIN)
        else:
            cs.render_bwd(st.pruned, st.cam, v, st.rec, st.pair_gid, st.tile_range,
                          st.img["t_final"], st.img["n_contrib"], dC, dD, dS, st.prm, st.cb,
                          cs.SKIP_CHAIN, grads=st.grads, ws=st.ws_bwd, tile_list=lst, max_tiles=T)
    res = {}
    for name, lst in [("plain", None)] + [(k, torch.cat([torch.tensor([T], device=dev), o]).int())
                                           for k, o in orders.items()]:
        ts = []
        for _ in range(25):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run(lst)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000)
        res[name] = statistics.median(ts[5:])
    print({k: round(x, 1) for k, x in res.items()}, "tile len mean/max", float(ln.float().mean()), int(ln.max()))


if __name__ == "__main__":
    main()
