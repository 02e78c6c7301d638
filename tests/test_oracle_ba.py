"""Pins for the NEXT-4 oracle (-m "not gpu"): the patch global-BA loss of
P:212-215 (reading R30) checked against closed forms, a library
routine (np.corrcoef), invariants and float64 central differences."""
import numpy as np
import pytest

C1, C2 = 0.01 ** 2, 0.03 ** 2


def images(rng, H=24, W=32):
    col = rng.uniform(0, 1, (3, H, W))
    dep = rng.uniform(0.5, 4, (H, W))
    oc = np.float32(np.clip(col + rng.normal(0, 0.1, col.shape), 0, 1))
    od = np.float32(dep * (1 + rng.normal(0, 0.05, dep.shape)))
    od[rng.uniform(size=od.shape) < 0.2] = 0.0  # invalid depth observations
    return col, dep, oc, od


def total(loss3, lam_d=1.0, lam_s=0.2):
    return loss3[0] + lam_d * loss3[1] + lam_s * (1.0 - loss3[2])


def test_identical_images_give_unit_ssim_and_zero_gradient(orc):
    rng = np.random.default_rng(0)
    col, dep, _, _ = images(rng)
    oc, od = np.float32(col), np.float32(dep)
    col, dep = np.float64(oc), np.float64(od)      # exactly representable pair
    patches = np.array([0, 5, 9, 11], dtype=np.int32)
    (dC, dD, dS), l3 = orc.ba_patch_loss(col, dep, oc, od, patches, n_rays=64 * 4, n_valid=256)
    assert l3[0] == 0.0 and l3[1] == 0.0
    assert l3[2] == pytest.approx(1.0, abs=1e-12)
    assert np.abs(dC).max() < 1e-12 and np.abs(dD).max() == 0.0 and np.abs(dS).max() == 0.0


def test_constant_patch_closed_form(orc):
    """x = a, y = b on a patch: variances and covariance vanish, so
    SSIM = (2ab + C1) / (a^2 + b^2 + C1) per channel."""
    H, W = 16, 16
    a = np.array([0.2, 0.5, 0.9]); b = np.array([0.25, 0.1, 0.9])
    col = np.ones((3, H, W)) * a[:, None, None]
    oc = np.float32(np.ones((3, H, W)) * b[:, None, None])
    dep = np.ones((H, W)); od = np.float32(np.ones((H, W)))
    (dC, _, _), l3 = orc.ba_patch_loss(col, dep, oc, od, np.array([3], np.int32), 64, 64)
    bb = np.float64(np.float32(b))
    want = np.mean((2 * a * bb + C1) / (a * a + bb * bb + C1))
    assert l3[2] == pytest.approx(want, rel=1e-12)
    assert l3[0] == pytest.approx(np.sum((a - bb) ** 2), rel=1e-12)   # 64 rays, N = 64


def test_structure_term_is_pearson_correlation(orc):
    """C1 = C2 = 0 and y with the mean and variance of x: SSIM = corr(x, y)."""
    rng = np.random.default_rng(3)
    H, W = 8, 8
    x = rng.uniform(0.2, 0.8, (3, H, W))
    y = rng.uniform(0.2, 0.8, (3, H, W))
    y = (y - y.mean(axis=(1, 2), keepdims=True)) / y.std(axis=(1, 2), keepdims=True)
    y = y * x.std(axis=(1, 2), keepdims=True) + x.mean(axis=(1, 2), keepdims=True)
    y32 = np.float32(y)
    # re-match the moments of x to the float32 y (the oracle reads y as float32)
    y64 = np.float64(y32)
    x = (x - x.mean(axis=(1, 2), keepdims=True)) / x.std(axis=(1, 2), keepdims=True)
    x = x * y64.std(axis=(1, 2), keepdims=True) + y64.mean(axis=(1, 2), keepdims=True)
    dep = np.ones((H, W)); od = np.float32(dep)
    _, l3 = orc.ba_patch_loss(x, dep, y32, od, np.array([0], np.int32), 64, 64, c1=0.0, c2=0.0)
    corr = np.mean([np.corrcoef(x[c].ravel(), y64[c].ravel())[0, 1] for c in range(3)])
    assert l3[2] == pytest.approx(corr, rel=1e-10)


def test_ssim_symmetric(orc):
    rng = np.random.default_rng(4)
    col, dep, oc, od = images(rng)
    col32 = np.float32(col)
    pt = np.array([1, 7, 10], np.int32)
    _, la = orc.ba_patch_loss(np.float64(col32), dep, oc, od, pt, 192, 100)
    _, lb = orc.ba_patch_loss(np.float64(oc), dep, col32, od, pt, 192, 100)
    assert la[2] == pytest.approx(lb[2], rel=1e-12)
    assert la[0] == pytest.approx(lb[0], rel=1e-12)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gradient_matches_central_differences(orc, seed):
    rng = np.random.default_rng(seed)
    col, dep, oc, od = images(rng)
    H, W = dep.shape
    pt = np.array([0, 6, 8, 11], np.int32)          # 4 of the 12 blocks of 32x24
    n_rays, n_valid = 64 * 6, 301                    # a sample larger than this keyframe's share
    (dC, dD, dS), l3 = orc.ba_patch_loss(col, dep, oc, od, pt, n_rays, n_valid)
    assert np.all(dS == 0)
    bw = W // 8
    inpatch = np.zeros((H, W), bool)
    for b in pt:
        by, bx = divmod(int(b), bw)
        inpatch[8 * by:8 * by + 8, 8 * bx:8 * bx + 8] = True
    assert np.all(dC[:, ~inpatch] == 0) and np.all(dD[~inpatch] == 0)
    h = 1e-6
    for _ in range(40):
        y, x = rng.integers(0, H), rng.integers(0, W)
        if not inpatch[y, x]:
            continue
        c = rng.integers(0, 3)
        cp = col.copy(); cp[c, y, x] += h
        cm = col.copy(); cm[c, y, x] -= h
        fd = (total(orc.ba_patch_loss(cp, dep, oc, od, pt, n_rays, n_valid)[1]) -
              total(orc.ba_patch_loss(cm, dep, oc, od, pt, n_rays, n_valid)[1])) / (2 * h)
        assert dC[c, y, x] == pytest.approx(fd, rel=1e-5, abs=1e-9)
        dp = dep.copy(); dp[y, x] += h
        dm = dep.copy(); dm[y, x] -= h
        fd = (total(orc.ba_patch_loss(col, dp, oc, od, pt, n_rays, n_valid)[1]) -
              total(orc.ba_patch_loss(col, dm, oc, od, pt, n_rays, n_valid)[1])) / (2 * h)
        assert dD[y, x] == pytest.approx(fd, rel=1e-5, abs=1e-9)
        if od[y, x] == 0:
            assert dD[y, x] == 0.0


def test_shares_add_up_over_keyframes(orc):
    """Splitting the sample over keyframes: the per-keyframe shares sum to the
    loss of the whole sample (normalisers are sample-wide)."""
    rng = np.random.default_rng(5)
    col, dep, oc, od = images(rng)
    pt = np.array([0, 2, 4, 6, 9], np.int32)
    _, whole = orc.ba_patch_loss(col, dep, oc, od, pt, 320, 200)
    _, a = orc.ba_patch_loss(col, dep, oc, od, pt[:2], 320, 200)
    _, b = orc.ba_patch_loss(col, dep, oc, od, pt[2:], 320, 200)
    np.testing.assert_allclose(a + b, whole, rtol=1e-12)


def test_count_valid(orc):
    od = np.zeros((16, 24), np.float32)
    od[0, 0] = 1.0; od[9, 9] = 2.0; od[15, 23] = 3.0; od[3, 12] = -1.0
    assert orc.ba_count_valid([od, od], [np.array([0, 4]), np.array([5])], 24) == 3
