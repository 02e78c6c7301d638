"""A/B timing of the C2 hot kernels for library variants (tools/variants.py):
`python tools/ab.py name1 name2 ...` runs each variant in its own process,
interleaved over `--rounds` rounds, and prints per variant the median (over
rounds) of each part's median launch time in us (512 MB L2 flush before every
launch): the backward kernel alone (CSPLAT_SKIP_CHAIN), the forward, the
stand-alone bin stage, the fused projection + bucket pass, and the
render-only graph (warm L2).  `base` = the in-tree libcsplat.so."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(reps):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2403_11247_b200 import csplat as cs
    from paper_2403_11247_b200.pipeline import RenderStep
    from scenes import synth

    dev = torch.device("cuda:0")
    sc = synth.replica_scene(0)
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    v = sc.views[0]
    st.size_pairs(v)
    H, W = sc.cam["height"], sc.cam["width"]
    st.set_upstream(*(torch.tensor(a, device=dev)
                      for a in synth.upstream(np.random.default_rng(1), H, W)))
    st.step(v)
    torch.cuda.synchronize()
    flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)

    def timed(fn, n=reps, do_flush=True, pre=None):
        ts = []
        for _ in range(n):
            if pre:
                pre()
            if do_flush:
                flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000)
        return statistics.median(ts[3:])

    res = {}
    res["bwd"] = timed(lambda: st.backward(v, flags=cs.SKIP_CHAIN | cs.WS_ZEROED),
                       pre=lambda: st.ws_bwd.zero_())
    res["fwd"] = timed(st.forward)
    res["bin"] = timed(lambda: cs.bin_tiles(st.rec, st.count, st.cam, st.capacity, ws=st.ws_bin,
                                    out=dict(pair_gid=st.pair_gid, tile_range=st.tile_range,
                                             n_pairs_dev=st.n_pairs), sync=False))
    res["projbin"] = timed(lambda: cs.project_bin(
        st.pruned, st.cam, v, st.capacity, st.prm, st.cb, rec=st.rec, count=st.count,
        ws=st.ws_bin, out=dict(pair_gid=st.pair_gid, tile_range=st.tile_range,
                               n_pairs_dev=st.n_pairs), sync=False))
    g = st.capture(v, render_only=True)
    res["render_only"] = timed(g.replay, do_flush=False)
    print(json.dumps(res))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    rounds = 3
    reps = 40
    for a in sys.argv[1:]:
        if a.startswith("--rounds="):
            rounds = int(a.split("=")[1])
        if a.startswith("--reps="):
            reps = int(a.split("=")[1])
    out = {v: [] for v in args}
    for _ in range(rounds):
        for v in args:
            env = dict(os.environ)
            if v != "base":
                env["CSPLAT_LIB"] = os.path.join(ROOT, "variants", v + ".so")
            p = subprocess.run([sys.executable, __file__, "--child", f"--reps={reps}"], env=env,
                               capture_output=True, text=True, timeout=600)
            line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
            if not line:
                print(v, "FAILED", p.stderr[-2000:])
                continue
            out[v].append(json.loads(line[-1]))
    for v, rs in out.items():
        if rs:
            print(v, {k: round(statistics.median(r[k] for r in rs), 1) for k in rs[0]})


if __name__ == "__main__":
    if "--child" in sys.argv:
        child(int([a for a in sys.argv if a.startswith("--reps=")][0].split("=")[1]))
    else:
        main()
