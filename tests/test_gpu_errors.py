"""The §8(b) error contract on the GPU (-m gpu): capacity overflow without a
host synchronisation (device status word, cut tiles left empty so the
renderers early-out, exact lists everywhere else), out-of-range codebook
indices (culled, status bit), the status slot collecting many calls, and the
window driver's capacity check over every keyframe."""
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


def _mid(env, seed=3):
    cs, dev = env["cs"], env["dev"]
    sc = synth.mid_scene(seed)
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    return sc, g


@pytest.mark.parametrize("fused", [False, True])
def test_capacity_overflow_status_word(env, fused):
    """No CSPLAT_SYNC: the call returns OK, the status slot gets
    STATUS_CAPACITY and the true total, every tile whose list fits is exact
    (oracle), every cut tile is empty, and the forward renders cut tiles as
    background."""
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    sc, g = _mid(env)
    cam, v = sc.cam, sc.views[0]
    S = orc.Scene(**sc.planes())
    rec_o, cnt_o = orc.project(S, cam, v)
    gid_o, rng_o = orc.bin_tiles(rec_o, cnt_o, cam)
    total = len(gid_o)
    cap = total // 2
    if fused:
        rec, cnt, b = cs.project_bin(g, cam, v, cap, sync=False)
    else:
        rec, cnt = cs.project(g, cam, v)
        b = cs.bin_tiles(rec, cnt, cam, capacity=cap, sync=False)
    torch.cuda.synchronize()
    slot = cs.range_status(b["tile_range"]).cpu().numpy().view(np.uint32)
    assert slot[0] & cs.STATUS_CAPACITY and slot[1] == total
    assert int(b["n_pairs_dev"].item()) == total
    rng = b["tile_range"][:-1].cpu().numpy().view(np.uint32)
    fits = rng_o[:, 1] <= cap
    assert fits.any() and (~fits).any()
    assert np.array_equal(rng[fits], rng_o[fits])
    assert np.all(rng[~fits, 0] == rng[~fits, 1])         # cut tiles: empty
    gid = b["pair_gid"].cpu().numpy().view(np.uint32) & cs.PAIR_GID_MASK
    for t in np.nonzero(fits)[0]:
        s, e = rng_o[t]
        assert np.array_equal(gid[s:e], gid_o[s:e])
    out = cs.render_fwd(rec, b["pair_gid"], b["tile_range"], cam)
    fo = orc.render_fwd(rec_o, gid_o, rng_o, cam)
    tx, ty = cs.tiles(cam)
    H, W = cam["height"], cam["width"]
    tile_of = (np.arange(H)[:, None] // 16) * tx + np.arange(W)[None, :] // 16
    ok = fits[tile_of] & (fo["flags"] == 0)
    assert np.abs(out["sil"].cpu().numpy() - fo["sil"])[ok].max() <= 1e-4
    cut = ~fits[tile_of]
    assert not out["sil"].cpu().numpy()[cut].any()
    assert bool((out["t_final"].cpu()[torch.from_numpy(cut)] == 1).all())
    # with CSPLAT_SYNC the same call reports CSPLAT_ERR_CAPACITY to the host
    with pytest.raises(cs.CsplatError, match="capacity"):
        cs.bin_tiles(rec, cnt, cam, capacity=cap, sync=True)


def test_status_slot_collects_calls(env):
    """The library only ORs / maxes into the status slot: one slot spans many
    asynchronous calls until the caller clears it."""
    torch, cs, dev = env["torch"], env["cs"], env["dev"]
    sc, g = _mid(env)
    rec, cnt = cs.project(g, sc.cam, sc.views[0])
    total = int(cnt.sum().item())
    out = None
    for cap in (total + 100, total // 3, total + 100):       # one overflowing call of three
        out = cs.bin_tiles(rec, cnt, sc.cam, capacity=cap, sync=False, out=None if out is None else
                           dict(out, pair_gid=torch.empty(cap, dtype=torch.int32, device=dev)))
    slot = cs.range_status(out["tile_range"]).cpu().numpy().view(np.uint32)
    assert slot[0] == cs.STATUS_CAPACITY and slot[1] == total
    cs.clear_status(out["tile_range"])
    cs.bin_tiles(rec, cnt, sc.cam, capacity=total, sync=False, out=out)
    slot = cs.range_status(out["tile_range"]).cpu().numpy().view(np.uint32)
    assert slot[0] == 0 and slot[1] == total


def test_out_of_range_code_index_culled_with_status(env):
    """Indices >= P: the Gaussian is culled (zero record, count 0, as the oracle
    does), the codebook's status word gets STATUS_CODE_INDEX, and every other
    record stays bit-exact."""
    torch, cs, orc, dev = env["torch"], env["cs"], env["orc"], env["dev"]
    sc = synth.tiny_scene(2)
    cb = sc.codebook
    si, _ = orc.rvq_assign(sc.log_scale, cb["scale_codes"])
    ri, _ = orc.rvq_assign(sc.quat, cb["rot_codes"])
    P = cb["scale_codes"].shape[1]
    S = orc.Scene(**sc.planes())
    _, cnt0 = orc.project(S, sc.cam, synth.IDENTITY_VIEW,
                          codebook=dict(cb, scale_idx=si, rot_idx=ri))
    live = np.nonzero(cnt0 > 0)[0]
    si[1, live[0]] = P
    ri[0, live[1]] = P + 7
    rec_o, cnt_o = orc.project(S, sc.cam, synth.IDENTITY_VIEW,
                               codebook=dict(cb, scale_idx=si, rot_idx=ri))
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    dt = torch.uint8
    cbt = cs.CodebookT(torch.tensor(cb["scale_codes"], device=dev),
                       torch.tensor(cb["rot_codes"], device=dev),
                       torch.tensor(si.astype(np.uint8), dtype=dt, device=dev),
                       torch.tensor(ri.astype(np.uint8), dtype=dt, device=dev), status=status)
    g = cs.GaussianMap.from_numpy(sc.planes(), device=dev)
    rec, cnt = cs.project(g, sc.cam, synth.IDENTITY_VIEW, cb=cbt)
    assert np.array_equal(rec.cpu().numpy().view(np.uint32), rec_o)
    assert np.array_equal(cnt.cpu().numpy(), cnt_o)
    assert int(status.item()) == cs.STATUS_CODE_INDEX
    # a valid codebook leaves the word untouched
    status.zero_()
    cbt.scale_idx[1, live[0]] = 0
    cbt.rot_idx[0, live[1]] = 0
    cs.project(g, sc.cam, synth.IDENTITY_VIEW, cb=cbt)
    assert int(status.item()) == 0


def test_window_capacity_check_covers_every_keyframe(env):
    """The window driver checks the status slots of BOTH view slots: an
    overflow on any keyframe of the iteration is reported, not only the last."""
    torch, cs, dev = env["torch"], env["cs"], env["dev"]
    from paper_2403_11247_b200.pipeline import RenderStep
    sc = synth.window_scene(0, n=20000, n_keyframes=4)
    st = RenderStep(sc.planes(), sc.cam, sc.codebook, device=dev)
    worst = st.size_pairs(sc.views[0], views=sc.views[1:])
    assert st.check_capacity() <= st.capacity
    a = st.view_slot()
    # overflow only on the first slot's view, then a fitting render on slot 0
    st._alloc_pairs(max(1, worst // 4))
    a._alloc_pairs(st.capacity * 8)
    st.prepare()
    a.project_bin(sc.views[1])          # slot a: fits
    st.project_bin(sc.views[0])         # slot 0: overflows
    with pytest.raises(cs.CsplatError, match="capacity"):
        st.check_capacity(slots=[st, a])
