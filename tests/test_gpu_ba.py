"""NEXT-4 GPU parity (-m gpu): the patch global BA (reading R30)
through the C ABI against the oracle -- active-tile binning bit-exact, the
valid-depth count exact, the loss and its upstream gradients, and one whole BA
iteration over several keyframes (gradients rel-L2 <= 1e-3)."""
import numpy as np
import pytest

from scenes import synth

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-3
GROUPS = ["mean", "opacity", "rgb", "log_scale", "quat", "mask"]


@pytest.fixture(scope="module")
def env():
    import torch
    import oracle
    from paper_2403_11247_b200 import _build, csplat
    _build.build()
    oracle.build()
    assert torch.cuda.is_available()
    return dict(torch=torch, cs=csplat, orc=oracle, dev=torch.device("cuda:0"))


def _observed(env, sc, view, seed):
    """Observed images: the oracle render at the view, perturbed (seeded)."""
    orc = env["orc"]
    rec, cnt = orc.project(orc.Scene(**sc.planes()), sc.cam, view)
    gid, rng = orc.bin_tiles(rec, cnt, sc.cam)
    fo = orc.render_fwd(rec, gid, rng, sc.cam)
    r = np.random.default_rng(seed)
    oc = np.float32(np.clip(fo["color"] + r.normal(0, 0.05, fo["color"].shape), 0, 1))
    od = np.float32(fo["depth"] * (1 + r.normal(0, 0.02, fo["depth"].shape)))
    od[r.uniform(size=od.shape) < 0.1] = 0.0
    return oc, od


def _active_tiles(patches, cam):
    tx = (cam["width"] + 15) // 16
    bw = cam["width"] // 8
    return sorted({(int(b) // bw * 8 // 16) * tx + (int(b) % bw) * 8 // 16 for b in patches})


def test_ba_patches_and_active_binning(env):
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    sc = synth.mid_scene(11)
    cam = sc.cam
    oc, od = _observed(env, sc, sc.views[0], 1)
    pt = synth.sample_patches(3, 1, cam["width"], cam["height"], 64 * 25)[0]
    pt_d = torch.tensor(pt, device=dev)
    mask, nv = cs.ba_patches(torch.tensor(od, device=dev), cam, pt_d)
    assert int(nv.item()) == orc.ba_count_valid([od], [pt], cam["width"])
    act = _active_tiles(pt, cam)
    bits = mask.cpu().numpy().view(np.uint32)
    got = [t for t in range(len(bits) * 32) if (bits[t >> 5] >> (t & 31)) & 1]
    assert got == act
    # csplat_bin_tiles_active == the oracle lists of the active tiles only
    S = orc.Scene(**sc.planes())
    rec_o, cnt_o = orc.project(S, cam, sc.views[0])
    gid_o, rng_o = orc.bin_tiles(rec_o, cnt_o, cam)
    keep_gid, keep_rng, pos = [], np.zeros_like(rng_o), 0
    for t in range(rng_o.shape[0]):
        seg = gid_o[rng_o[t, 0]:rng_o[t, 1]] if t in set(act) else gid_o[:0]
        keep_gid.append(seg)
        keep_rng[t] = (pos, pos + len(seg))
        pos += len(seg)
    keep_gid = np.concatenate(keep_gid)
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    rec, cnt = cs.project(g, cam, sc.views[0])
    b = cs.bin_tiles(rec, cnt, cam, capacity=len(gid_o) + 64, tile_active=mask)
    n = int(b["n_pairs_dev"].item())
    assert n == len(keep_gid) and n < len(gid_o)
    assert np.array_equal(b["pair_gid"][:n].cpu().numpy().view(np.uint32) & cs.PAIR_GID_MASK,
                          keep_gid)
    assert np.array_equal(b["tile_range"][:-1].cpu().numpy().view(np.uint32), keep_rng)


def test_ba_patch_loss_parity(env):
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    sc = synth.mid_scene(12)
    cam = sc.cam
    oc, od = _observed(env, sc, sc.views[0], 2)
    view = synth.perturbed_view(np.random.default_rng(5), rot_deg=1.0, trans=0.02)
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    rec, cnt = cs.project(g, cam, view)
    b = cs.bin_tiles(rec, cnt, cam, capacity=int(cnt.sum().item()) + 64)
    img = cs.render_fwd(rec, b["pair_gid"], b["tile_range"], cam)
    pt = synth.sample_patches(4, 2, cam["width"], cam["height"], 64 * 60)[0]
    n_rays = 64 * 60                        # this keyframe holds part of the sample
    ocd, odd = torch.tensor(oc, device=dev), torch.tensor(od, device=dev)
    pt_d = torch.tensor(pt, device=dev)
    _, nv = cs.ba_patches(odd, cam, pt_d)
    nv.add_(17)                             # other keyframes' valid rays
    (dC, dD, dS), l3 = cs.ba_patch_loss(img, ocd, odd, cam, pt_d, n_rays, nv,
                                        lambda_depth=0.7, lambda_ssim=0.3)
    (rC, rD, rS), rl = orc.ba_patch_loss(img["color"].double().cpu().numpy(),
                                         img["depth"].double().cpu().numpy(), oc, od, pt, n_rays,
                                         int(nv.item()), lambda_d=0.7, lambda_s=0.3)
    np.testing.assert_allclose(l3.cpu().numpy(), rl, rtol=2e-5, atol=1e-7)
    for a, r in ((dC, rC), (dD, rD), (dS, rS)):
        a = a.double().cpu().numpy()
        assert np.abs(a - r).max() <= 1e-5 * max(np.abs(r).max(), 1e-6)


@pytest.mark.parametrize("seed,driver", [(0, "pipelined"), (1, "pipelined"), (0, "batched"),
                                         (1, "batched")])
def test_ba_iteration_parity(env, seed, driver):
    """One BA iteration over 4 keyframes (RenderStep: prune -> project ->
    active bin -> fwd -> loss -> bwd ACCUMULATE) against the oracle's sum of
    per-keyframe gradients on the pruned map; per-keyframe pose gradients."""
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    from paper_2403_11247_b200.ba import BatchedBA, ba_loss_value, gpu_ba
    from paper_2403_11247_b200.pipeline import RenderStep
    sc = synth.mid_scene(20 + seed)
    cam = sc.cam
    rng = np.random.default_rng(seed)
    views = [sc.views[0]] + [synth.perturbed_view(rng, 2.0, 0.03) for _ in range(3)]
    obs = [_observed(env, sc, v, 10 + i) for i, v in enumerate(views)]
    # the observed images come from a slightly different pose: a non-trivial loss
    rviews = [synth.perturbed_view(np.random.default_rng(50 + i), 0.5, 0.01) @
              np.vstack([v, [0, 0, 0, 1]]) for i, v in enumerate(views)]
    rviews = [np.float32(v) for v in rviews]
    patches = synth.sample_patches(seed, len(views), cam["width"], cam["height"], 64 * 48)
    # drop patches holding a pixel whose float32/float64 termination is ambiguous
    keep = sc.mask > orc.mask_tau(0.01)
    pl = {k: v[..., keep] for k, v in sc.planes().items()}
    S = orc.Scene(**pl)
    ref = []
    for k, v in enumerate(rviews):
        rec_o, cnt_o = orc.project(S, cam, v)
        gid_o, rng_o = orc.bin_tiles(rec_o, cnt_o, cam)
        fo = orc.render_fwd(rec_o, gid_o, rng_o, cam)
        bw = cam["width"] // 8
        good = [b for b in patches[k]
                if not fo["flags"][8 * (b // bw):8 * (b // bw) + 8, 8 * (b % bw):8 * (b % bw) + 8].any()]
        patches[k] = np.array(good, dtype=np.int32)
        ref.append((rec_o, gid_o, rng_o, fo))
    n_rays = 64 * sum(len(p) for p in patches)
    n_valid = orc.ba_count_valid([o[1] for o in obs], patches, cam["width"])
    tot = np.zeros(3)
    go_sum, poses_o = None, []
    for k, v in enumerate(rviews):
        rec_o, gid_o, rng_o, fo = ref[k]
        (rC, rD, rS), l3 = orc.ba_patch_loss(fo["color"], fo["depth"], obs[k][0], obs[k][1],
                                             patches[k], n_rays, n_valid)
        tot += l3
        go = orc.render_bwd(S, cam, v, rec_o, gid_o, rng_o, rC, rD, rS)
        poses_o.append(go["pose"])
        go_sum = go if go_sum is None else {n: go_sum[n] + go[n] for n in GROUPS}
    # GPU
    st = RenderStep(sc.planes(), cam, None, device=dev)
    st.size_pairs(rviews[0], views=rviews[1:])
    oc = [torch.tensor(o[0], device=dev) for o in obs]
    od = [torch.tensor(o[1], device=dev) for o in obs]
    if driver == "batched":  # one multi-view front, tile-list renders, one chain over views
        ba = BatchedBA(st, rviews, oc, od, patches, rank=0, world=1)
    else:
        ba = gpu_ba(st, rviews, oc, od, patches, rank=0, world=1)
    ba.run()
    torch.cuda.synchronize()
    assert ba.n_rays == n_rays and int(ba.n_valid.item()) == n_valid
    np.testing.assert_allclose(ba.loss3.cpu().numpy(), tot, rtol=1e-4, atol=1e-7)
    assert ba_loss_value(ba.loss3) == pytest.approx(ba_loss_value(tot), rel=1e-4)
    kk = int(st.n_kept.item())
    for name in GROUPS:
        a = st.grads[name].double().cpu().numpy().reshape(-1, st.n)[:, :kk].reshape(-1)
        r = go_sum[name].reshape(-1)
        assert np.linalg.norm(a - r) / np.linalg.norm(r) <= GRAD_TOL, name
    for k in range(len(views)):
        a = ba.poses[k].double().cpu().numpy()
        assert np.linalg.norm(a - poses_o[k]) / np.linalg.norm(poses_o[k]) <= GRAD_TOL


def test_ba_edge_cases(env):
    """Keyframes without patches, patch ids outside the image's whole blocks
    (ignored), an image whose width / height are not multiples of 8, and an
    empty sample."""
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    sc = synth.mid_scene(13, width=150, height=100)     # 18 x 12 whole 8x8 blocks
    cam = sc.cam
    oc, od = _observed(env, sc, sc.views[0], 3)
    ocd, odd = torch.tensor(oc, device=dev), torch.tensor(od, device=dev)
    bw, bh = cam["width"] // 8, cam["height"] // 8
    good = np.array([0, bw - 1, bw * (bh - 1), bw * bh - 1, 37], np.int32)
    bad = np.array([-1, bw * bh, 10 ** 6], np.int32)
    pt = torch.tensor(np.concatenate([good, bad]), device=dev)
    mask, nv = cs.ba_patches(odd, cam, pt)
    assert int(nv.item()) == orc.ba_count_valid([od], [good], cam["width"])
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    rec, cnt = cs.project(g, cam, sc.views[0])
    b = cs.bin_tiles(rec, cnt, cam, capacity=int(cnt.sum().item()) + 64, tile_active=mask)
    img = cs.render_fwd(rec, b["pair_gid"], b["tile_range"], cam)
    n_rays = 64 * len(good)
    (dC, dD, dS), l3 = cs.ba_patch_loss(img, ocd, odd, cam, pt, n_rays, nv)
    (rC, rD, rS), rl = orc.ba_patch_loss(img["color"].double().cpu().numpy(),
                                         img["depth"].double().cpu().numpy(), oc, od, good,
                                         n_rays, int(nv.item()))
    np.testing.assert_allclose(l3.cpu().numpy(), rl, rtol=2e-5, atol=1e-7)
    assert np.abs(dC.double().cpu().numpy() - rC).max() <= 1e-5 * max(np.abs(rC).max(), 1e-6)
    # an empty sample: zero upstream, untouched loss, an all-clear tile mask
    l0 = torch.zeros(3, device=dev)
    empty = torch.zeros(0, dtype=torch.int32, device=dev)
    m0, nv0 = cs.ba_patches(odd, cam, empty)
    assert int(nv0.item()) == 0 and int(m0.abs().sum().item()) == 0
    (eC, eD, eS), l0 = cs.ba_patch_loss(img, ocd, odd, cam, empty, 64, nv0, loss3=l0)
    assert float(eC.abs().sum()) == 0 and float(eD.abs().sum()) == 0 and float(l0.abs().sum()) == 0
    b0 = cs.bin_tiles(rec, cnt, cam, capacity=64, tile_active=m0)
    assert int(b0["n_pairs_dev"].item()) == 0
