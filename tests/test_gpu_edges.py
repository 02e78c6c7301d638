"""Edge cases of the C ABI on the GPU (-m gpu): empty inputs, a device-side
count of zero, a 1x1 image, non-finite attributes, and the error contract."""
import math

import numpy as np
import pytest

from scenes import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import oracle
    from paper_2403_11247_b200 import _build, csplat
    _build.build()
    oracle.build()
    return dict(torch=torch, cs=csplat, orc=oracle, dev=torch.device("cuda:0"))


def empty_map(torch, cs, dev, n=0):
    z = lambda *s: torch.zeros(s, device=dev)
    return cs.GaussianMap(mean=z(3, n), opacity=z(n), rgb=z(3, n), log_scale=z(3, n),
                          quat=z(4, n), mask=z(n))


def test_empty_map_full_path(env):
    torch, cs, dev = env["torch"], env["cs"], env["dev"]
    cam = synth.CAMERAS["tiny"]
    g = empty_map(torch, cs, dev)
    rec, cnt = cs.project(g, cam, synth.IDENTITY_VIEW)
    b = cs.bin_tiles(rec, cnt, cam, capacity=0)
    assert int(b["n_pairs_dev"].item()) == 0
    assert not b["tile_range"].any()
    out = cs.render_fwd(rec, b["pair_gid"], b["tile_range"], cam)
    assert not out["color"].any() and not out["sil"].any() and not out["n_contrib"].any()
    assert bool((out["t_final"] == 1).all())
    H, W = cam["height"], cam["width"]
    gr = cs.render_bwd(g, cam, synth.IDENTITY_VIEW, rec, b["pair_gid"], b["tile_range"],
                       out["t_final"], out["n_contrib"], torch.ones((3, H, W), device=dev),
                       torch.ones((H, W), device=dev), torch.ones((H, W), device=dev))
    assert not gr["pose"].any()
    pr, _, km, nk = cs.mask_prune(g)
    assert int(nk.item()) == 0
    idx, rc = cs.rvq_assign(torch.zeros((3, 0), device=dev), torch.zeros((2, 4, 3), device=dev))
    (dC, dD, dS), l3 = cs.tracking_loss(out, out["color"], out["depth"])
    assert not dC.any() and float(l3[0].item()) == 0.0


def test_zero_device_count(env):
    """n_dev = 0: every Gaussian beyond the device count is treated as absent."""
    torch, cs, dev = env["torch"], env["cs"], env["dev"]
    sc = synth.tiny_scene(0)
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    g.n_dev = torch.zeros(1, dtype=torch.int64, device=dev)
    rec, cnt = cs.project(g, sc.cam, sc.views[0])
    assert not cnt.any() and not rec.any()
    idx = torch.full((2, g.n), 7, dtype=torch.uint8, device=dev)
    cs.rvq_assign(g.log_scale, torch.tensor(sc.codebook["scale_codes"], device=dev),
                  n_dev=g.n_dev, idx=idx, want_recon=False)
    assert bool((idx == 7).all())          # nothing written beyond n_dev
    pr, _, km, nk = cs.mask_prune(g, keep_map=torch.empty(g.n, dtype=torch.int32, device=dev))
    assert int(nk.item()) == 0 and bool((km == -1).all())


def test_one_pixel_image(env):
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    cam = dict(fx=10.0, fy=10.0, cx=0.0, cy=0.0, width=1, height=1, near=0.01, far=100.0)
    n = 5
    mean = np.float32([[0, 0.01, -0.01, 0, 0], [0, 0, 0.01, -0.02, 0], [1, 1.5, 2, 2.5, 3]])
    S = dict(mean=mean, opacity=np.float32([0, 1, -1, 2, 0.5]), rgb=np.full((3, n), 0.5, np.float32),
             log_scale=np.full((3, n), math.log(0.05), np.float32),
             quat=np.tile(np.float32([[1], [0], [0], [0]]), (1, n)), mask=np.full(n, 3, np.float32))
    g = cs.GaussianMap.from_numpy(S, device=dev)
    rec, cnt = cs.project(g, cam, synth.IDENTITY_VIEW)
    rec_o, cnt_o = orc.project(orc.Scene(**S), cam, synth.IDENTITY_VIEW)
    assert np.array_equal(rec.cpu().numpy().view(np.uint32), rec_o)
    gid_o, rng_o = orc.bin_tiles(rec_o, cnt_o, cam)
    b = cs.bin_tiles(rec, cnt, cam, capacity=16)
    out = cs.render_fwd(rec, b["pair_gid"], b["tile_range"], cam)
    fo = orc.render_fwd(rec_o, gid_o, rng_o, cam)
    assert abs(float(out["sil"][0, 0]) - fo["sil"][0, 0]) < 1e-5


def test_non_finite_attributes_are_culled(env):
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    sc = synth.tiny_scene(2)
    sc.mean[0, 5] = np.nan
    sc.log_scale[1, 6] = np.inf
    sc.quat[:, 7] = 0.0                    # zero quaternion
    sc.opacity[8] = np.nan
    sc.rgb[2, 9] = -np.inf
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    rec, cnt = cs.project(g, sc.cam, sc.views[0])
    rec_o, cnt_o = orc.project(orc.Scene(**sc.planes()), sc.cam, sc.views[0])
    assert np.array_equal(rec.cpu().numpy().view(np.uint32), rec_o)
    assert not cnt[5:10].any()


def test_error_contract(env):
    torch, cs, dev = env["torch"], env["cs"], env["dev"]
    sc = synth.tiny_scene(0)
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    bad = dict(sc.cam, fx=-1.0)
    with pytest.raises(cs.CsplatError, match="invalid argument"):
        cs.project(g, bad, sc.views[0])
    rec, cnt = cs.project(g, sc.cam, sc.views[0])
    with pytest.raises(cs.CsplatError, match="workspace"):
        cs.bin_tiles(rec, cnt, sc.cam, capacity=1000,
                     ws=torch.empty(8, dtype=torch.uint8, device=dev))
    mis = torch.empty(g.n * 16 + 1, dtype=torch.int32, device=dev)[1:].view(g.n, 16)
    with pytest.raises(cs.CsplatError, match="misaligned"):
        cs.project(g, sc.cam, sc.views[0], rec=mis)
