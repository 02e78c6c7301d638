"""Pins for the CPU oracle (-m "not gpu"): the oracle checked against what the
paper and mathematics fix -- worked examples (tests/golden), closed forms,
invariants, brute force and float64 finite differences.  Nothing here compares
the oracle with itself or with the CUDA path."""
import json
import math
import os

import numpy as np
import pytest

from scenes import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def one_gaussian_scene(orc, means, sigma=0.1, o_hat=0.8, quats=None, scales=None, rgb=None,
                       mask=3.0):
    means = np.asarray(means, dtype=np.float64).reshape(-1, 3)
    n = means.shape[0]
    ls = np.full((3, n), math.log(sigma)) if scales is None else np.log(np.asarray(scales)).T
    q = np.tile([[1.0], [0], [0], [0]], (1, n)) if quats is None else np.asarray(quats).T
    o = np.full(n, math.log(o_hat / (1 - o_hat)))
    c = np.ones((3, n)) * 0.5 if rgb is None else np.asarray(rgb).T
    return orc.Scene(mean=np.float32(means.T), opacity=np.float32(o), rgb=np.float32(c),
                     log_scale=np.float32(ls), quat=np.float32(q),
                     mask=np.full(n, mask, dtype=np.float32))


CF_CAM = dict(fx=48.0, fy=48.0, cx=32.0, cy=24.0, width=64, height=48, near=0.01, far=100.0)
IDV = synth.IDENTITY_VIEW


def sigma_prime_from_rec(rec, dil=0.3):
    f = rec.view(np.float32)
    ca, cb, cc = float(f[2]), float(f[3]) / 2, float(f[4])
    Q = np.array([[ca, cb], [cb, cc]], dtype=np.float64)
    return np.linalg.inv(Q) - dil * np.eye(2)


# ---------------------------------------------------------------- DA helpers

def test_pexp_accuracy(orc):
    xs = np.linspace(-86.0, 88.0, 20001, dtype=np.float32)
    xs = np.concatenate([xs, np.float32([0.0, -0.0, 1e-8, -1e-8, 0.5, -0.5])])
    worst = 0.0
    for x in xs:
        ref = math.exp(float(x))
        got = orc.pexp(float(x))
        worst = max(worst, abs(got - ref) / ref)
    assert orc.pexp(0.0) == 1.0
    assert worst < 3.0 * 2.0 ** -23, worst       # within ~1.5 ulp of float32


def test_plog_accuracy(orc):
    xs = np.concatenate([np.linspace(1.0001, 255.0, 20001, dtype=np.float32),
                         np.float32([2.0, 4.0, 204.0, 255.0, 1.5, math.sqrt(2)])])
    for x in xs:
        ref = math.log(float(x))
        got = orc.plog(float(x))
        assert abs(got - ref) <= 4e-7 * max(1.0, abs(ref)) + 2e-8, (x, got, ref)
    assert abs(orc.plog(204.0) * 2 - GOLD["projection"]["on_axis"]["k2"]) < 2e-6


def test_mask_threshold_worked_examples(orc):
    for case in GOLD["mask"]["cases"]:
        tau = orc.mask_tau(case["eps"])
        assert int(case["m"] > tau) == case["M"]
        if "dM_dm" in case:
            s = 1 / (1 + math.exp(-case["m"]))
            assert abs(s * (1 - s) - case["dM_dm"]) < 1e-12


def test_mask_threshold_exact_near_tau(orc):
    """Every float32 within 1e-3 of tau: the DA test m > fl32(tau) equals the
    real-number test Sig(m) > 0.01 (exact logit in float64)."""
    tau = np.float32(orc.mask_tau(0.01))
    exact = math.log(0.01 / 0.99)
    lo, hi = np.float32(tau - 1e-3), np.float32(tau + 1e-3)
    m = lo
    n = 0
    while m <= hi:
        assert (m > tau) == (float(m) > exact)
        m = np.nextafter(m, np.float32(np.inf))
        n += 1
    assert n > 4000
    assert not (tau > tau)       # sig(m) = eps is masked (R12)


# ---------------------------------------------------------------- projection

def test_projection_closed_form(orc):
    g = GOLD["projection"]
    sc = one_gaussian_scene(orc, [g["on_axis"]["mean"], g["off_axis"]["mean"]])
    rec, cnt = orc.project(sc, CF_CAM, IDV)
    f = rec.view(np.float32)
    for i, key in enumerate(["on_axis", "off_axis"]):
        ref = g[key]
        assert np.allclose(f[i, :2], ref["uv"], atol=1e-5)
        assert np.allclose(sigma_prime_from_rec(rec[i]) + 0.3 * np.eye(2), ref["sigma_prime"],
                           rtol=1e-5, atol=1e-5)
    assert abs(f[0, 6] - g["on_axis"]["k2"]) < 2e-6
    px0, py0 = rec[0, 12] & 0xFFFF, rec[0, 12] >> 16
    px1, py1 = rec[0, 13] & 0xFFFF, rec[0, 13] >> 16
    assert [px0, px1] == g["on_axis"]["pixel_rect"]["x"]
    assert [py0, py1] == g["on_axis"]["pixel_rect"]["y"]
    # tiles: x 24..40 -> tiles 1..2, y 16..32 -> tiles 1..2
    assert cnt[0] == 4


def test_projection_covariance_examples(orc):
    """S:58-60 through the on-axis projection: Sigma' = (f/z)^2 Sigma_xy."""
    cam = dict(CF_CAM)
    z = 40.0
    for case in GOLD["covariance"]["cases"]:
        sc = one_gaussian_scene(orc, [[0, 0, z]], quats=[case["quat_wxyz"]],
                                scales=[np.array(case["scale"]) * 0.5], o_hat=0.99)
        rec, cnt = orc.project(sc, cam, IDV)
        sp = sigma_prime_from_rec(rec[0]) / (cam["fx"] / z) ** 2 / 0.25
        assert np.allclose(sp, case["sigma_xy"], atol=2e-5), (sp, case)


def _rot_from_quat(q):
    from scipy.spatial.transform import Rotation
    w, x, y, z = q
    return Rotation.from_quat([x, y, z, w]).as_matrix()


def test_projection_numeric_jacobian(orc):
    """Sigma' against J_num W Sigma W^T J_num^T with J_num the central-difference
    Jacobian of the pinhole map and R from scipy (independent of the oracle)."""
    rng = np.random.default_rng(3)
    cam = dict(fx=300.0, fy=310.0, cx=160.0, cy=120.0, width=320, height=240, near=0.01,
               far=100.0)
    view = synth.perturbed_view(rng, rot_deg=10, trans=0.2)
    n = 40
    z = rng.uniform(2, 6, n)
    uv = np.stack([rng.uniform(20, 300, n), rng.uniform(20, 220, n)])
    pc = np.stack([(uv[0] - cam["cx"]) / cam["fx"] * z, (uv[1] - cam["cy"]) / cam["fy"] * z, z])
    Rv, tv = view[:, :3].astype(np.float64), view[:, 3].astype(np.float64)
    mean = Rv.T @ (pc - tv[:, None])
    scales = np.exp(rng.normal(-3, 0.5, (n, 3)))
    quats = rng.standard_normal((n, 4))
    sc = one_gaussian_scene(orc, mean.T, quats=quats, scales=scales, o_hat=0.9)
    rec, cnt = orc.project(sc, cam, view)
    def proj(p):
        return np.array([cam["fx"] * p[0] / p[2] + cam["cx"], cam["fy"] * p[1] / p[2] + cam["cy"]])
    for i in range(n):
        assert cnt[i] > 0
        mu = sc.mean[:, i].astype(np.float64)
        p = Rv @ mu + tv
        Jn = np.zeros((2, 3))
        for k in range(3):
            e = np.zeros(3); e[k] = 1e-5 * p[2]
            Jn[:, k] = (proj(p + e) - proj(p - e)) / (2 * e[k])
        R = _rot_from_quat(sc.quat[:, i].astype(np.float64) / np.linalg.norm(sc.quat[:, i]))
        Sig = R @ np.diag(np.exp(2 * sc.log_scale[:, i].astype(np.float64))) @ R.T
        ref = Jn @ Rv @ Sig @ Rv.T @ Jn.T
        got = sigma_prime_from_rec(rec[i])
        assert np.allclose(got, ref, rtol=2e-3, atol=2e-4 * np.abs(ref).max()), (i, got, ref)
        assert np.allclose(rec[i, :2].view(np.float32), proj(p), atol=2e-3)


def test_projection_depth_doubling(orc):
    """doubling z with isotropic Sigma quarters Sigma' (minus dilation)."""
    a = one_gaussian_scene(orc, [[0, 0, 2.0], [0, 0, 4.0]], sigma=0.1)
    rec, _ = orc.project(a, CF_CAM, IDV)
    s1, s2 = sigma_prime_from_rec(rec[0]), sigma_prime_from_rec(rec[1])
    assert np.allclose(s2 * 4, s1, rtol=1e-5)


def test_projection_culls(orc):
    sc = one_gaussian_scene(orc, [[0, 0, 2], [0, 0, -1], [0, 0, 200], [100, 0, 2], [0, 0, 2],
                                  [0, 0, 2]])
    sc.mask[4] = -10.0                         # masked (Eq 6-7)
    sc.opacity[5] = -30.0                      # o = 0: 255 o <= 1 (R2)
    rec, cnt = orc.project(sc, CF_CAM, IDV)
    assert list(cnt > 0) == [True, False, False, False, False, False]
    assert (rec[1:] == 0).all()


# ---------------------------------------------------------------- binning

def test_binning_bruteforce(orc):
    for sc in (synth.tiny_scene(0), synth.mid_scene(1, n=800)):
        S = orc.Scene(**sc.planes())
        rec, cnt = orc.project(S, sc.cam, sc.views[0])
        gid, rng_ = orc.bin_tiles(rec, cnt, sc.cam)
        tx, ty = orc.tiles(sc.cam)
        pairs = []
        for i in np.nonzero(cnt)[0]:
            x0, y0 = rec[i, 12] & 0xFFFF, rec[i, 12] >> 16
            x1, y1 = rec[i, 13] & 0xFFFF, rec[i, 13] >> 16
            for t in range(tx * ty):
                bx0, by0 = (t % tx) * 16, (t // tx) * 16
                if x0 <= bx0 + 15 and x1 >= bx0 and y0 <= by0 + 15 and y1 >= by0:
                    pairs.append((t, int(rec[i, 7]), int(i)))
        pairs.sort()
        assert len(pairs) == cnt.sum() == len(gid)
        assert [p[2] for p in pairs] == list(gid)
        assert rng_[0, 0] == 0 and rng_[-1, 1] == len(gid)
        assert (rng_[1:, 0] == rng_[:-1, 1]).all()
        for t in range(tx * ty):
            assert rng_[t, 1] - rng_[t, 0] == sum(1 for p in pairs if p[0] == t)


# ---------------------------------------------------------------- forward

def render_all(orc, S, cam, view=IDV, prm=None, codebook=None):
    rec, cnt = orc.project(S, cam, view, prm, codebook)
    gid, rng_ = orc.bin_tiles(rec, cnt, cam)
    return rec, cnt, gid, rng_, orc.render_fwd(rec, gid, rng_, cam, prm)


def test_forward_closed_form_alpha(orc):
    g = GOLD["alpha"]
    for key, mean in (("on_axis_pixels", [0, 0, 2]), ("off_axis_pixels", [0.5, 0, 2])):
        S = one_gaussian_scene(orc, [mean], rgb=[[1.0, 0.25, 0.5]])
        _, _, _, _, out = render_all(orc, S, CF_CAM)
        for p in g[key]:
            a = out["sil"][p["py"], p["px"]]
            assert abs(a - p["alpha"]) < g["tolerance"], (p, a)
            assert abs(out["depth"][p["py"], p["px"]] - 2.0 * a) < 2 * g["tolerance"]
            assert np.allclose(out["color"][:, p["py"], p["px"]], np.array([1, 0.25, 0.5]) * a,
                               atol=g["tolerance"])


def test_forward_two_gaussians(orc):
    g = GOLD["two_gaussians"]
    o_back = 20.0
    S = orc.Scene(mean=np.float32([[0, 0], [0, 0], [1, 2]]), opacity=np.float32([0.0, o_back]),
                  rgb=np.float32([[1, 0], [0, 1], [0, 0]]),
                  log_scale=np.float32(np.full((3, 2), math.log(0.05))),
                  quat=np.float32([[1, 1], [0, 0], [0, 0], [0, 0]]), mask=np.float32([3, 3]))
    for mode in ("smooth", "default"):
        ref = g[mode]
        prm = orc.params(alpha_max=ref["alpha_max"], t_min=ref["t_min"])
        _, _, _, _, out = render_all(orc, S, CF_CAM, prm=prm)
        tol = g["tolerance"] if mode == "default" else 1e-6
        assert np.allclose(out["color"][:, 24, 32], ref["color"], atol=tol)
        assert abs(out["depth"][24, 32] - ref["depth"]) < tol
        assert abs(out["sil"][24, 32] - ref["sil"]) < tol
        if "t_final" in ref:
            assert abs(out["t_final"][24, 32] - ref["t_final"]) < tol


def test_forward_empty_and_invariants(orc):
    cam = synth.CAMERAS["tiny"]
    S = one_gaussian_scene(orc, np.zeros((0, 3)))
    _, _, gid, _, out = render_all(orc, S, cam)
    assert len(gid) == 0 and not out["color"].any() and not out["sil"].any()
    for seed in range(4):
        sc = synth.mid_scene(seed, n=600, width=96, height=64)
        S = orc.Scene(**sc.planes())
        rec, cnt, gid, rng_, out = render_all(orc, S, sc.cam)
        assert out["sil"].min() >= 0 and out["sil"].max() <= 1
        assert np.abs(out["sil"] - (1 - out["t_final"])).max() < 1e-9
        # a transparent Gaussian (o -> 0) changes nothing
        S2 = orc.Scene(**{k: np.concatenate([getattr(S, k), v], axis=-1) for k, v in dict(
            mean=np.float32([[0], [0], [2]]), opacity=np.float32([-30]),
            rgb=np.float32([[1], [1], [1]]), log_scale=np.float32([[-1], [-1], [-1]]),
            quat=np.float32([[1], [0], [0], [0]]), mask=np.float32([3])).items()})
        out2 = render_all(orc, S2, sc.cam)[-1]
        for k in ("color", "depth", "sil", "t_final"):
            assert np.array_equal(out[k], out2[k])


def test_forward_equal_depth_permutation(orc):
    """permuting identical Gaussians at equal depth changes nothing."""
    base = one_gaussian_scene(orc, [[0.1, 0, 2], [0.1, 0, 2], [-0.1, 0.05, 2.5]],
                              rgb=[[1, 0, 0], [1, 0, 0], [0, 1, 0]], o_hat=0.6)
    perm = one_gaussian_scene(orc, [[-0.1, 0.05, 2.5], [0.1, 0, 2], [0.1, 0, 2]],
                              rgb=[[0, 1, 0], [1, 0, 0], [1, 0, 0]], o_hat=0.6)
    a = render_all(orc, base, CF_CAM)[-1]
    b = render_all(orc, perm, CF_CAM)[-1]
    for k in ("color", "depth", "sil"):
        assert np.array_equal(a[k], b[k])


def test_forward_tiled_equals_untiled(orc):
    """The tiled renderer reaches the per-pixel brute-force definition exactly."""
    sc = synth.tiny_scene(0)
    S = orc.Scene(**sc.planes())
    rec, cnt, gid, rng_, out = render_all(orc, S, sc.cam)
    H, W = sc.cam["height"], sc.cam["width"]
    for py in range(H):
        for px in range(W):
            o6, _ = orc.render_pixel(rec, cnt, sc.cam, px, py)
            ref = [out["color"][0, py, px], out["color"][1, py, px], out["color"][2, py, px],
                   out["depth"][py, px], out["sil"][py, px], out["t_final"][py, px]]
            assert np.array_equal(o6, ref), (px, py)
    sc = synth.mid_scene(2)
    S = orc.Scene(**sc.planes())
    rec, cnt, gid, rng_, out = render_all(orc, S, sc.cam)
    r = np.random.default_rng(0)
    for _ in range(150):
        px, py = int(r.integers(0, sc.cam["width"])), int(r.integers(0, sc.cam["height"]))
        o6, _ = orc.render_pixel(rec, cnt, sc.cam, px, py)
        assert np.array_equal(o6[:5], [out["color"][0, py, px], out["color"][1, py, px],
                                       out["color"][2, py, px], out["depth"][py, px],
                                       out["sil"][py, px]])


def test_forward_masked_removal_invariance(orc):
    """a masked Gaussian renders as invisible -- removing it
    changes no output bit."""
    sc = synth.tiny_scene(1)
    S = orc.Scene(**sc.planes())
    out = render_all(orc, S, sc.cam)[-1]
    keep = sc.mask > orc.mask_tau(0.01)
    S2 = orc.Scene(**{k: v[..., keep] for k, v in sc.planes().items()})
    out2 = render_all(orc, S2, sc.cam)[-1]
    for k in ("color", "depth", "sil", "t_final", "n_contrib"):
        assert np.array_equal(out[k], out2[k])


def test_forward_depth_tie_lowest_index_first(orc):
    sc = synth.tiny_scene(0)
    S = orc.Scene(**sc.planes())
    rec, cnt, gid, rng_, _ = render_all(orc, S, sc.cam)
    assert rec[0, 7] == rec[1, 7]
    pos = {}
    for t in range(rng_.shape[0]):
        lst = list(gid[rng_[t, 0]:rng_[t, 1]])
        if 0 in lst and 1 in lst:
            pos[t] = lst.index(0) < lst.index(1)
    assert pos and all(pos.values())


# ---------------------------------------------------------------- backward

GROUPS = ["mean", "opacity", "rgb", "log_scale", "quat", "mask"]


def _fd_grads(orc, sc, wC, wD, wS, clamp=False):
    cam, v = sc.cam, sc.views[0]
    S = orc.Scene(**{k: v_.copy() for k, v_ in sc.planes().items()})

    def L(xi=None):
        c, d, s = orc.smooth_render(S, cam, v, xi=xi, clamp=clamp)
        return (wC * c).sum() + (wD * d).sum() + (wS * s).sum()

    out = {}
    for name in GROUPS:
        a2 = getattr(S, name).reshape(-1, S.n)
        fd = np.zeros(a2.shape)
        for k in range(a2.shape[0]):
            for i in range(S.n):
                x0 = a2[k, i]
                h = 1e-3 * max(1.0, abs(float(x0)))
                xp, xm = np.float32(x0 + h), np.float32(x0 - h)
                a2[k, i] = xp; lp = L()
                a2[k, i] = xm; lm = L()
                a2[k, i] = x0
                fd[k, i] = (lp - lm) / (float(xp) - float(xm))
        out[name] = fd
    fdp = np.zeros(6)
    for k in range(6):
        e = np.zeros(6); e[k] = 1e-6
        fdp[k] = (L(e) - L(-e)) / 2e-6
    out["pose"] = fdp
    return out


@pytest.mark.parametrize("seed", list(range(10)))
def test_backward_finite_differences(orc, seed):
    """Smooth-mode analytic gradient (mean, opacity, rgb, log-scale, quaternion,
    mask STE, pose) = float64 central differences."""
    sc = synth.small_fd_scene(seed)
    r = np.random.default_rng(100 + seed)
    H, W = sc.cam["height"], sc.cam["width"]
    wC, wD, wS = r.standard_normal((3, H, W)), r.standard_normal((H, W)), r.standard_normal((H, W))
    S = orc.Scene(**sc.planes())
    an = orc.smooth_bwd(S, sc.cam, sc.views[0], wC, wD, wS)
    fd = _fd_grads(orc, sc, wC, wD, wS)
    for k in GROUPS + ["pose"]:
        a, f = an[k].reshape(-1), fd[k].reshape(-1)
        err = np.linalg.norm(a - f) / np.linalg.norm(f)
        assert err < 1e-4, (k, err)


def test_backward_finite_differences_jacobian_clamp(orc):
    """The J clamp branch (R6): Gaussians outside the 1.3x FOV, FD-checked."""
    sc = synth.small_fd_scene(0)
    sc.mean[0] += np.linspace(-3.0, 3.0, sc.n).astype(np.float32)
    r = np.random.default_rng(7)
    H, W = sc.cam["height"], sc.cam["width"]
    wC, wD, wS = r.standard_normal((3, H, W)), r.standard_normal((H, W)), r.standard_normal((H, W))
    S = orc.Scene(**sc.planes())
    an = orc.smooth_bwd(S, sc.cam, sc.views[0], wC, wD, wS, clamp=True)
    fd = _fd_grads(orc, sc, wC, wD, wS, clamp=True)
    for k in GROUPS + ["pose"]:
        a, f = an[k].reshape(-1), fd[k].reshape(-1)
        assert np.linalg.norm(a - f) / np.linalg.norm(f) < 1e-4, k


def test_backward_zero_upstream(orc):
    sc = synth.mid_scene(0, n=500, width=64, height=48)
    S = orc.Scene(**sc.planes())
    rec, cnt, gid, rng_, out = render_all(orc, S, sc.cam)
    H, W = sc.cam["height"], sc.cam["width"]
    g = orc.render_bwd(S, sc.cam, sc.views[0], rec, gid, rng_, np.zeros((3, H, W)),
                       np.zeros((H, W)), np.zeros((H, W)))
    for k in GROUPS + ["pose"]:
        assert not np.any(g[k])


def test_backward_closed_form_red(orc):
    """dLoss/dc_red for a single centred Gaussian, smooth and capped."""
    g = GOLD["backward_red"]
    for mode, o_logit, amax in (("smooth", 30.0, 1.0), ("capped", 30.0, 0.99)):
        S = orc.Scene(mean=np.float32([[0], [0], [2]]), opacity=np.float32([o_logit]),
                      rgb=np.float32([[0.5], [0.2], [0.2]]),
                      log_scale=np.float32([[math.log(0.05)]] * 3),
                      quat=np.float32([[1], [0], [0], [0]]), mask=np.float32([3]))
        prm = orc.params(alpha_max=amax, t_min=0.0)
        rec, cnt, gid, rng_, out = render_all(orc, S, CF_CAM, prm=prm)
        H, W = 48, 64
        dC = np.zeros((3, H, W)); dC[0, 24, 32] = 2 * (out["color"][0, 24, 32] - 1)
        gr = orc.render_bwd(S, CF_CAM, IDV, rec, gid, rng_, dC, np.zeros((H, W)),
                            np.zeros((H, W)), prm=prm)
        assert abs(gr["rgb"][0, 0] - g[mode]) < 1e-9
        if mode == "capped":           # R23: no gradient through a capped alpha
            assert gr["opacity"][0, 0] == 0.0


# ---------------------------------------------------------------- R-VQ

def _rvq_bruteforce(x, codes):
    """Exhaustive float64 argmin on the float32 DA residual, per stage."""
    L, P, d = codes.shape
    n = x.shape[1]
    idx = np.zeros((L, n), dtype=np.int64)
    sh = np.zeros((d, n), dtype=np.float32)
    near_tie = np.zeros(n, dtype=bool)
    for l in range(L):
        r = (x - sh) if l else x.copy()
        dist = ((codes[l].astype(np.float64)[:, :, None] - r.astype(np.float64)[None]) ** 2).sum(1)
        best = dist.argmin(0)
        srt = np.sort(dist, axis=0)
        gap = (srt[1] - srt[0]) / np.maximum(srt[0], 1e-30) if P > 1 else np.inf
        near_tie |= gap < 1e-5
        idx[l] = best
        sh = codes[l][best].T.astype(np.float32) if l == 0 else (sh + codes[l][best].T).astype(np.float32)
    return idx, sh, near_tie


def test_rvq_bruteforce(orc):
    sc = synth.room_scene(4000, synth.CAMERAS["scannet"], 5, codebook_LP=(4, 64))
    for x, codes in ((sc.log_scale, sc.codebook["scale_codes"]), (sc.quat, sc.codebook["rot_codes"])):
        idx, recon = orc.rvq_assign(x, codes)
        bidx, bsh, tie = _rvq_bruteforce(x, codes)
        ok = ~tie
        assert ok.mean() > 0.99
        assert (idx[:, ok] == bidx[:, ok]).all()
        assert np.array_equal(recon[:, ok], bsh[:, ok])


def test_rvq_special_cases(orc):
    r = np.random.default_rng(0)
    x = r.standard_normal((3, 50)).astype(np.float32)
    # L = P = 1: forced choice, recon = the code
    idx, rec = orc.rvq_assign(x, np.float32([[[0.3, -0.2, 0.1]]]))
    assert (idx == 0).all() and np.allclose(rec, np.float32([[0.3], [-0.2], [0.1]]))
    # exact-match cascade: stage 1 holds the inputs, stage 2 only zeros
    codes = np.zeros((2, 50, 3), dtype=np.float32)
    codes[0] = x.T
    idx, rec = orc.rvq_assign(x, codes)
    assert (idx[0] == np.arange(50)).all() and (idx[1] == 0).all()
    assert np.array_equal(rec, x)
    # duplicate codes -> lowest index (R11)
    codes = r.standard_normal((1, 8, 3)).astype(np.float32)
    codes[0, 6] = codes[0, 2]
    xx = codes[0, [2]].T.copy()
    idx, _ = orc.rvq_assign(xx, codes)
    assert idx[0, 0] == 2
    # decode = sum of selected codes
    ex = GOLD["rvq"]["decode_example"]
    codes = np.float32([[ex["codes"][0]], [ex["codes"][1]]])
    idx, rec = orc.rvq_assign(np.float32([[5], [5], [5]]), codes)
    assert np.array_equal(rec[:, 0], np.float32(ex["sum"]))
    # L = 1 is plain VQ (nearest code)
    codes = r.standard_normal((1, 16, 3)).astype(np.float32)
    idx, _ = orc.rvq_assign(x, codes)
    d = ((codes[0][:, :, None] - x[None]) ** 2).sum(1)
    assert (idx[0] == d.argmin(0)).all()


# ---------------------------------------------------------------- R-VQ update (NEXT-2)

def test_rvq_update_degenerate_and_centroids(orc):
    """N identical vectors, L = 1 -> the assigned code becomes
    that vector and a second round has zero loss; two separated clusters with
    P = 2 -> codes = the cluster centroids, loss = within-cluster scatter."""
    v = np.float32([[0.3], [-1.2], [2.0]])
    x = np.repeat(v, 8, axis=1)
    codes = np.random.default_rng(0).standard_normal((1, 8, 3)).astype(np.float32)
    idx, _ = orc.rvq_assign(x, codes)
    new, cnt, loss = orc.rvq_update(x, codes, idx)
    assert cnt.sum() == 8 and np.array_equal(new[0, idx[0, 0]], v[:, 0])
    assert loss[0] > 0
    new2, _, loss2 = orc.rvq_update(x, new, orc.rvq_assign(x, new)[0])
    assert loss2[0] == 0.0 and loss2[1] == 0.0
    r = np.random.default_rng(1)
    a = r.normal(0, 0.1, (3, 50)) + np.array([[5.0], [0], [0]])
    b = r.normal(0, 0.1, (3, 70)) - np.array([[5.0], [0], [0]])
    x = np.concatenate([a, b], 1).astype(np.float32)
    codes = np.float32([[[4.0, 0, 0], [-4.0, 0, 0]]])
    idx, _ = orc.rvq_assign(x, codes)
    new, cnt, loss = orc.rvq_update(x, codes, idx)
    assert list(cnt[0]) == [50, 70]
    assert np.allclose(new[0, 0], a.astype(np.float32).mean(1), atol=1e-6)
    assert np.allclose(new[0, 1], b.astype(np.float32).mean(1), atol=1e-6)
    scatter = sum(((c.astype(np.float32).astype(np.float64) - cc[:, None]) ** 2).sum()
                  for c, cc in ((a, codes[0, 0]), (b, codes[0, 1])))
    assert abs(loss[0] - scatter) < 1e-6 * scatter
    assert abs(loss[1] - scatter / (120 * 2)) < 1e-9


def test_rvq_update_decreases_reconstruction_error(orc):
    """Lloyd iterations (assign, update) never increase the stage-1 error, and
    the stage losses of a trained cascade decrease across stages."""
    sc = synth.room_scene(3000, synth.CAMERAS["tum"], 2, codebook_LP=(3, 32))
    x, codes = sc.log_scale, sc.codebook["scale_codes"].copy()
    prev = np.inf
    for _ in range(6):
        idx, _ = orc.rvq_assign(x, codes)
        codes, _, loss = orc.rvq_update(x, codes, idx)
        assert loss[0] <= prev * (1 + 1e-9)
        prev = loss[0]
    idx, _ = orc.rvq_assign(x, codes)
    _, _, loss = orc.rvq_update(x, codes, idx)
    assert loss[0] > loss[1] > loss[2]


# ---------------------------------------------------------------- window mask schedule (NEXT-3)

def test_mask_loss_worked_examples(orc):
    """SPEC S:219-221 (Eq 8): all m = 0 -> 0.5; m -> -inf -> 0; {0, 20} -> 0.75;
    the gradient is Sig'(m)/N_a and only in-frustum Gaussians count."""
    L, d = orc.mask_loss(np.zeros(6), np.ones(6))
    assert abs(L - 0.5) < 1e-12 and np.allclose(d, 0.25 / 6)
    L, _ = orc.mask_loss(np.full(3, -80.0), np.ones(3))
    assert L < 1e-30
    L, _ = orc.mask_loss(np.float32([0, 20]), np.ones(2))
    assert abs(L - 0.75) < 1e-8
    L, d = orc.mask_loss(np.float32([0, 20, -3]), np.uint8([1, 1, 0]), lam=2.0)
    assert abs(L - 0.75) < 1e-8 and d[2] == 0.0 and abs(d[0] - 2 * 0.25 / 2) < 1e-12


def test_keyframe_overlap_worked_examples(orc):
    """candidate = current pose -> (almost) all points; facing the
    opposite way -> 0; translated by half the scene -> strictly between."""
    cam = dict(fx=60.0, fy=60.0, cx=39.5, cy=29.5, width=80, height=60, near=0.01, far=100.0)
    depth = np.random.default_rng(0).uniform(2, 4, (60, 80)).astype(np.float32)
    depth[::5] = 0.0                                  # invalid rows are not counted
    valid = int((depth > 0).sum())
    I = synth.IDENTITY_VIEW
    back = synth.look_view((0, 0, 0), -np.pi / 2)      # looking along -z
    shifted = I.copy(); shifted[0, 3] = -1.5           # camera moved +1.5 m in x
    counts = orc.keyframe_overlap(depth, cam, I, [I, back, shifted])
    # border pixels sit exactly on the frustum boundary, where float32 rounding decides
    assert counts[0] >= 0.97 * valid and counts[0] <= valid
    assert counts[1] == 0
    assert 0 < counts[2] < counts[0]


# ---------------------------------------------------------------- tracking loss (NEXT-1)

def test_tracking_loss_worked_example(orc):
    g = GOLD["tracking_loss"]
    C = np.zeros((3, 2, 2)); C[0] = g["color_r"]
    (dC, dD, dS), loss, flags = orc.tracking_loss(C, np.array(g["depth"]), np.array(g["sil"]),
                                                  np.zeros((3, 2, 2)), np.array(g["obs_depth"]))
    assert np.allclose(loss, [g["L_t"], g["L_c"], g["L_d"]], rtol=1e-12)
    assert np.allclose(dC[0], g["d_color_r"]) and not dC[1:].any()
    assert np.allclose(dD, g["d_depth"]) and not dS.any() and not flags.any()


def test_tracking_loss_gradient_fd(orc):
    """The returned upstream gradient is the derivative of the returned loss."""
    r = np.random.default_rng(5)
    H, W = 6, 7
    C, D = r.uniform(0, 1, (3, H, W)), r.uniform(0.5, 3, (H, W))
    S = np.where(r.uniform(0, 1, (H, W)) < 0.7, 0.999, 0.5)
    OC = r.uniform(0, 1, (3, H, W)).astype(np.float32)
    OD = np.where(r.uniform(0, 1, (H, W)) < 0.8, r.uniform(0.5, 3, (H, W)), 0).astype(np.float32)
    (dC, dD, _), loss, _ = orc.tracking_loss(C, D, S, OC, OD, lambda_d=0.7)
    h = 1e-6
    for arr, grad in ((C, dC), (D, dD)):
        flat, gflat = arr.reshape(-1), grad.reshape(-1)
        for i in r.choice(flat.size, 12, replace=False):
            x0 = flat[i]
            flat[i] = x0 + h; lp = orc.tracking_loss(C, D, S, OC, OD, lambda_d=0.7)[1][0]
            flat[i] = x0 - h; lm = orc.tracking_loss(C, D, S, OC, OD, lambda_d=0.7)[1][0]
            flat[i] = x0
            assert abs((lp - lm) / (2 * h) - gflat[i]) < 1e-6
    # flags mark silhouettes within 1e-5 of the gate
    (_, _, _), _, fl = orc.tracking_loss(C, D, np.full((H, W), 0.990005), OC, OD)
    assert fl.all()


# ---------------------------------------------------------------- prune

def test_prune_worked_example(orc):
    g = GOLD["prune"]
    n = g["n"]
    mask = np.full(n, 2.0, dtype=np.float32)
    mask[g["masked_indices"]] = g["masked_logit"]
    vals = np.arange(n, dtype=np.float32)
    outs, _, keep_map, k = orc.mask_prune([vals, mask], [], mask_plane=1)
    assert k == len(g["kept"]) and list(outs[0]) == g["kept"]
    assert [int(v) for v in keep_map] == [g["kept"].index(i) if i in g["kept"] else -1 for i in range(n)]
    outs2, _, _, k2 = orc.mask_prune(outs, [], mask_plane=1)
    assert k2 == k                    # second prune removes nothing


def test_prune_render_invariance(orc):
    """P:139 / S:254: rendering after pruning is bitwise the rendering before."""
    sc = synth.mid_scene(3, n=1500, width=96, height=64)
    sc.codebook = None
    names = ["mean", "opacity", "rgb", "log_scale", "quat", "mask"]
    planes, shapes = [], []
    for k in names:
        a = getattr(sc, k).reshape(-1, sc.n)
        shapes.append(a.shape[0])
        planes += list(a)
    mask_plane = sum(shapes[:5])
    outs, _, keep_map, k = orc.mask_prune(planes, [], mask_plane=mask_plane)
    assert k == int((sc.mask > orc.mask_tau(0.01)).sum())
    S = orc.Scene(**sc.planes())
    off, pr = 0, {}
    for name, c in zip(names, shapes):
        pr[name] = np.stack(outs[off:off + c]).reshape((c, k) if c > 1 else (k,))
        off += c
    S2 = orc.Scene(**pr)
    a = render_all(orc, S, sc.cam)[-1]
    b = render_all(orc, S2, sc.cam)[-1]
    for key in ("color", "depth", "sil", "t_final", "n_contrib"):
        assert np.array_equal(a[key], b[key])


# ---------------------------------------------------------------- round-2 pins
# (early termination / n_contrib, the DA J-clamp branch, keyframe
# overlap under a non-identity current pose)

def _gauss_list(orc, gs):
    means = np.array([g["mean"] for g in gs], dtype=np.float64)
    n = len(gs)
    return orc.Scene(mean=np.float32(means.T),
                     opacity=np.float32([math.log(g["o_hat"] / (1 - g["o_hat"])) for g in gs]),
                     rgb=np.float32(np.array([g["rgb"] for g in gs]).T),
                     log_scale=np.float32(np.array([[math.log(g["sigma"])] * 3 for g in gs]).T),
                     quat=np.float32(np.tile([[1.0], [0], [0], [0]], (1, n))),
                     mask=np.full(n, 3.0, dtype=np.float32))


def _check_pixel(out, px, py, ref, tol):
    assert np.allclose(out["color"][:, py, px], ref["color"], atol=tol), out["color"][:, py, px]
    assert abs(out["depth"][py, px] - ref["depth"]) < tol
    assert abs(out["sil"][py, px] - ref["sil"]) < tol
    assert abs(out["t_final"][py, px] - ref["t_final"]) < tol
    assert out["n_contrib"][py, px] == ref["n_contrib"]


def test_termination_alpha_max_one_drops_back_gaussian(orc):
    """SPEC S:147 with alpha_max = 1 and t_min = 1e-4 (R3): the back Gaussian's
    alpha is exactly 1, so T(1 - alpha) = 0 < t_min and it is NOT composited."""
    ref = GOLD["termination"]["alpha_max_1"]
    S = orc.Scene(mean=np.float32([[0, 0], [0, 0], [1, 2]]), opacity=np.float32([0.0, 20.0]),
                  rgb=np.float32([[1, 0], [0, 1], [0, 0]]),
                  log_scale=np.float32(np.full((3, 2), math.log(0.05))),
                  quat=np.float32([[1, 1], [0, 0], [0, 0], [0, 0]]), mask=np.float32([3, 3]))
    prm = orc.params(alpha_max=ref["alpha_max"], t_min=ref["t_min"])
    rec, cnt, gid, rng_, out = render_all(orc, S, CF_CAM, prm=prm)
    px, py = ref["pixel"]
    _check_pixel(out, px, py, ref, 1e-7)
    o6, ncomp = orc.render_pixel(rec, cnt, CF_CAM, px, py, prm)   # untiled form agrees
    assert ncomp == 1 and abs(o6[5] - ref["t_final"]) < 1e-7 and abs(o6[1]) < 1e-12


def test_termination_mid_list_n_contrib(orc):
    """R3 mid-list: a non-covering entry between two composited ones, then the
    terminating entry, then one never examined.  n_contrib counts list
    positions (last composited index + 1), not composited entries."""
    ref = GOLD["termination"]["mid_list"]
    S = _gauss_list(orc, ref["gaussians"])
    prm = orc.params(alpha_max=ref["alpha_max"], t_min=ref["t_min"])
    rec, cnt, gid, rng_, out = render_all(orc, S, CF_CAM, prm=prm)
    px, py = ref["pixel"]
    t = (py // 16) * ((64 + 15) // 16) + px // 16
    assert list(gid[rng_[t, 0]:rng_[t, 1]]) == [0, 1, 2, 3, 4]      # depth order
    _check_pixel(out, px, py, ref, ref["tolerance"])
    o6, ncomp = orc.render_pixel(rec, cnt, CF_CAM, px, py, prm)
    assert ncomp == ref["n_composited"]
    assert np.allclose(o6, list(ref["color"]) + [ref["depth"], ref["sil"], ref["t_final"]],
                       atol=ref["tolerance"])
    # without the terminating Gaussian, the fifth one is composited instead
    S2 = _gauss_list(orc, [g for i, g in enumerate(ref["gaussians"]) if i != 3])
    out2 = render_all(orc, S2, CF_CAM, prm=prm)[-1]
    assert out2["n_contrib"][py, px] == 4
    assert abs(out2["t_final"][py, px] - 0.001) < 1e-6


@pytest.mark.parametrize("case", ["x_clamped", "y_clamped"])
def test_projection_jacobian_clamp_closed_form(orc, case):
    """R6 in the DA projection (oracle_project): an off-FOV Gaussian's Sigma' is
    built from the clamped x/z (or y/z), its mean from the unclamped one."""
    g = GOLD["jacobian_clamp"]
    c = g[case]
    S = one_gaussian_scene(orc, [c["mean"]], sigma=g["sigma"], o_hat=g["o_hat"])
    rec, cnt = orc.project(S, CF_CAM, IDV)
    assert cnt[0] > 0
    f = rec[0].view(np.float32)
    assert abs(f[0] - c["uv"][0]) < 1e-4 and abs(f[1] - c["uv"][1]) < 1e-4
    Sp = sigma_prime_from_rec(rec[0], dil=0.0)          # Sigma' incl. the 0.3 I dilation
    ref = np.array(c["sigma_prime"])
    assert np.allclose(Sp, ref, rtol=g["tolerance_rel"], atol=1e-3), Sp
    px0, py0, px1, py1 = rec[0, 12] & 0xffff, rec[0, 12] >> 16, rec[0, 13] & 0xffff, rec[0, 13] >> 16
    assert [px0, px1] == c["pixel_rect"]["x"] and [py0, py1] == c["pixel_rect"]["y"]


def test_keyframe_overlap_plane_non_identity_pose(orc):
    """P:138 overlap count against closed-form counts on a fronto-parallel
    plane seen from a rotated and translated current camera."""
    from scipy.spatial.transform import Rotation
    k = GOLD["keyframe_overlap_plane"]
    cam = dict(k["camera"], near=0.01, far=100.0)
    R = Rotation.from_rotvec([0.3, -0.5, 0.2]).as_matrix()
    t = np.array([0.4, -0.7, 1.1])
    cur = np.concatenate([R, t[:, None]], 1).astype(np.float32)
    depth = np.full((cam["height"], cam["width"]), k["depth"], dtype=np.float32)
    names = ["shift_x", "shift_y", "forward", "behind"]
    views = []
    for nm in names:
        v = cur.astype(np.float64).copy()
        v[:, 3] += k["shifts"][nm]
        views.append(v.astype(np.float32))
    counts = orc.keyframe_overlap(depth, cam, cur, views + [cur])
    for i, nm in enumerate(names):
        assert counts[i] == k["counts"][nm], (nm, counts[i])
    # the current view itself: every interior pixel maps to itself; the border
    # pixels land exactly on the frustum boundary, where float32 rounding decides
    H, W = depth.shape
    assert (H - 2) * (W - 2) <= counts[-1] <= H * W


def test_out_of_range_code_index_culls(orc):
    """a Gaussian whose codebook index is >= P is culled -- its
    record is all zero, count 0 -- and nothing else changes: the render equals
    the render of the map without it (bit for bit)."""
    sc = synth.tiny_scene(2)
    cb = dict(sc.codebook)
    si, _ = orc.rvq_assign(sc.log_scale, cb["scale_codes"])
    ri, _ = orc.rvq_assign(sc.quat, cb["rot_codes"])
    P = cb["scale_codes"].shape[1]
    S = orc.Scene(**sc.planes())
    rec0, cnt0 = orc.project(S, sc.cam, IDV, codebook=dict(cb, scale_idx=si, rot_idx=ri))
    live = np.nonzero(cnt0 > 0)[0]
    bad = [int(live[0]), int(live[1])]
    si2, ri2 = si.copy(), ri.copy()
    si2[1, bad[0]] = P           # a later stage out of range
    ri2[0, bad[1]] = P + 7       # a rotation index out of range
    rec, cnt = orc.project(S, sc.cam, IDV, codebook=dict(cb, scale_idx=si2, rot_idx=ri2))
    assert (cnt[bad] == 0).all() and not rec[bad].any()
    others = np.setdiff1d(np.arange(sc.n), bad)
    assert np.array_equal(rec[others], rec0[others]) and np.array_equal(cnt[others], cnt0[others])
    keep = np.ones(sc.n, bool); keep[bad] = False
    S2 = orc.Scene(**{k: v[..., keep] for k, v in sc.planes().items()})
    cb2 = dict(cb, scale_idx=si[:, keep], rot_idx=ri[:, keep])
    a = render_all(orc, S, sc.cam, codebook=dict(cb, scale_idx=si2, rot_idx=ri2))[-1]
    b = render_all(orc, S2, sc.cam, codebook=cb2)[-1]
    for k in ("color", "depth", "sil", "t_final", "n_contrib"):
        assert np.array_equal(a[k], b[k])


def test_threads_do_not_change_results(orc):
    """The OpenMP build of the timed baseline: the forward, the
    projection and R-VQ are bit-identical at any thread count; the backward's
    per-thread float64 partials change only the summation order."""
    sc = synth.mid_scene(1)
    S = orc.Scene(**sc.planes())
    H, W = sc.cam["height"], sc.cam["width"]
    r = np.random.default_rng(3)
    up = r.standard_normal((3, H, W)), r.standard_normal((H, W)), r.standard_normal((H, W))
    res = []
    try:
        for th in (1, 4):
            orc.set_threads(th)
            rec, cnt, gid, rng_, out = render_all(orc, S, sc.cam)
            gr = orc.render_bwd(S, sc.cam, sc.views[0], rec, gid, rng_, *up)
            idx, rc = orc.rvq_assign(sc.log_scale, sc.codebook["scale_codes"])
            res.append((rec, out, gr, idx, rc))
    finally:
        orc.set_threads(1)
    (r1, o1, g1, i1, c1), (r4, o4, g4, i4, c4) = res
    assert np.array_equal(r1, r4) and np.array_equal(i1, i4) and np.array_equal(c1, c4)
    for k in ("color", "depth", "sil", "t_final", "n_contrib", "flags"):
        assert np.array_equal(o1[k], o4[k])
    for k in g1:
        assert np.allclose(g1[k], g4[k], rtol=1e-12, atol=1e-14), k


# ---------------------------------------------------------------- NEXT-2 (R-VQ training side)

def test_rvq_code_grad_closed_form_and_fd(orc):
    """STE (reading R31): S_hat = sum_l C^l[i^l] is linear in every code, so
    dL/dC^l[k] = sum of dL/dS_hat over the vectors whose stage-l index is k.
    Pinned by a hand example and by float64 central differences of
    L(C) = sum_n <w_n, S_hat_n(C)> with numpy's own decode."""
    # hand example: 3 vectors, L = 2, P = 2, d = 2
    idx = np.array([[0, 1, 0], [1, 1, 0]], np.uint16)
    g = np.array([[1.0, 2.0, 4.0], [10.0, 20.0, 40.0]])
    out = orc.rvq_code_grad(g, idx, 2, 2)
    assert np.array_equal(out[0], [[5.0, 50.0], [2.0, 20.0]])   # stage 0: {0,2} -> 0, {1} -> 1
    assert np.array_equal(out[1], [[4.0, 40.0], [3.0, 30.0]])   # stage 1: {2} -> 0, {0,1} -> 1
    # accumulate adds onto the given buffer
    out2 = orc.rvq_code_grad(g, idx, 2, 2, d_codes=out.copy())
    assert np.array_equal(out2, 2 * out)
    # FD on a random problem
    r = np.random.default_rng(4)
    L, P, d, n = 3, 8, 4, 200
    codes = r.standard_normal((L, P, d))
    idx = r.integers(0, P, (L, n)).astype(np.uint16)
    w = r.standard_normal((d, n))

    def loss(c):
        shat = sum(c[l][idx[l]] for l in range(L))       # [n, d]
        return float((shat.T * w).sum())
    an = orc.rvq_code_grad(w, idx, L, P)
    h = 1e-3
    fd = np.zeros_like(codes)
    for l in range(L):
        for k in range(P):
            for j in range(d):
                cp, cm = codes.copy(), codes.copy()
                cp[l, k, j] += h
                cm[l, k, j] -= h
                fd[l, k, j] = (loss(cp) - loss(cm)) / (2 * h)
    assert np.allclose(an, fd, rtol=1e-9, atol=1e-9)


def test_rvq_init_stage_fig4(orc):
    """Fig 4 (reading R32): stage 0's codes are the sampled vectors
    themselves; stage l's codes are the sampled vectors' stage-l residuals, so
    after the closest-code assignment every sampled vector sits at distance
    exactly 0 from its stage-l code (checked in numpy float32 from the
    oracle's codes and indices)."""
    r = np.random.default_rng(9)
    d, n, L, P = 4, 3000, 3, 32
    x = np.float32(r.standard_normal((d, n)) * [[1.0], [0.5], [0.25], [2.0]])
    codes = np.zeros((L, P, d), np.float32)
    idx = None
    samples = []
    for l in range(L):
        s = r.choice(n, P, replace=False)
        samples.append(s)
        codes = orc.rvq_init_stage(x, codes, l, idx, s)
        if l == 0:
            assert np.array_equal(codes[0], x[:, s].T)
        idx, _ = orc.rvq_assign(x, codes[:l + 1])
        idx = np.concatenate([idx, np.zeros((L - l - 1, n), np.uint16)])
    for l in range(L):
        s = samples[l]
        sh = np.zeros((d, P), np.float32)
        for m in range(l):
            sh = codes[m][idx[m, s]].T if m == 0 else np.float32(sh + codes[m][idx[m, s]].T)
        res = np.float32(x[:, s] - sh)                       # stage-l residuals (float32)
        assert np.array_equal(codes[l].T, res)             # the init copies them bit for bit
        c = codes[l][idx[l, s]].T
        assert not np.any(c - res), l                      # distance exactly 0
