"""Seeded synthetic scene generators shared by tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic: it only draws random
numbers (numpy PCG64, ``default_rng(seed)``) and lays them out in the ABI's
planar SoA layout.  Both the CUDA path and the CPU oracle consume what it
returns; neither is imported here.  Recipes follow DESIGN.md "Input recipe"
(SURVEY.md section 8(d) configs C1-C5).

Layouts (float32): mean [3,n], opacity logit [n], rgb [3,n], log_scale [3,n],
quat wxyz [4,n], mask logit [n].  Views are row-major 3x4 world->camera.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# mask logit threshold for eps = 0.01 rounded to float32 (Eq 6 reading R12);
# the generator only uses it to place adversarial test values next to it.
TAU_F32 = np.float32(math.log(0.01 / 0.99))

CAMERAS = {
    # C1 tiny; the closed-form pins use cx=32, cy=24 instead.
    "tiny": dict(fx=48.0, fy=48.0, cx=31.5, cy=23.5, width=64, height=48, near=0.01, far=100.0),
    # Replica-shaped 1200x680 ("1200x980" read as 1200x680, R25)
    "replica": dict(fx=600.0, fy=600.0, cx=599.5, cy=339.5, width=1200, height=680, near=0.01,
                    far=100.0),
    # TUM-RGBD fr1-shaped 640x480
    "tum": dict(fx=517.3, fy=516.5, cx=318.6, cy=255.3, width=640, height=480, near=0.01,
                far=100.0),
    # ScanNet-shaped 640x480
    "scannet": dict(fx=577.6, fy=578.7, cx=318.9, cy=242.7, width=640, height=480, near=0.01,
                    far=100.0),
}

IDENTITY_VIEW = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 1, 0]], dtype=np.float32)


@dataclass
class SynthScene:
    mean: np.ndarray
    opacity: np.ndarray
    rgb: np.ndarray
    log_scale: np.ndarray
    quat: np.ndarray
    mask: np.ndarray
    cam: dict
    views: list = field(default_factory=list)
    codebook: dict | None = None   # scale_codes [L,P,3], rot_codes [L,P,4]

    @property
    def n(self) -> int:
        return int(self.opacity.shape[0])

    def planes(self):
        return dict(mean=self.mean, opacity=self.opacity, rgb=self.rgb,
                    log_scale=self.log_scale, quat=self.quat, mask=self.mask)


def _unit_quats(rng, n):
    q = rng.standard_normal((4, n))
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    q[:, q[0] < 0] *= -1.0
    return q.astype(np.float32)


def _room_depth(rng, dirs, room, n_slabs):
    """Depth along z of each ray (dirs [3,n], z component 1) in a box room with
    fronto-parallel occluder slabs.  Returns z [n]."""
    hx, hy, zf = room
    dx, dy = dirs[0], dirs[1]
    with np.errstate(divide="ignore", invalid="ignore"):
        tx = np.where(np.abs(dx) > 1e-9, hx / np.abs(dx), np.inf)
        ty = np.where(np.abs(dy) > 1e-9, hy / np.abs(dy), np.inf)
    z = np.minimum(np.minimum(tx, ty), zf)
    for _ in range(n_slabs):
        zs = rng.uniform(1.5, 4.0)
        cxs, cys = rng.uniform(-0.6, 0.6) * zs, rng.uniform(-0.4, 0.4) * zs
        hxs, hys = rng.uniform(0.2, 0.8), rng.uniform(0.2, 0.8)
        xs, ys = dx * zs, dy * zs
        hit = (np.abs(xs - cxs) < hxs) & (np.abs(ys - cys) < hys) & (zs < z)
        z = np.where(hit, zs, z)
    return z


def room_scene(n, cam, seed, mask_keep=0.75, opacity_mu=3.0, opacity_sd=1.5, n_slabs=8,
               room=(3.0, 1.5, 5.0), codebook_LP=(4, 256)):
    """Replica/TUM/ScanNet-shaped scene: pixel-uniform back-projection into a
    box room plus occluder slabs."""
    rng = np.random.default_rng(seed)
    W, H = cam["width"], cam["height"]
    px = rng.uniform(0, W - 1, n)
    py = rng.uniform(0, H - 1, n)
    dirs = np.stack([(px - cam["cx"]) / cam["fx"], (py - cam["cy"]) / cam["fy"], np.ones(n)])
    z = _room_depth(rng, dirs, room, n_slabs) * (1.0 + rng.normal(0, 0.002, n))
    mean = (dirs * z).astype(np.float32)
    s_px = rng.lognormal(math.log(2.5), 0.35, (3, n))
    s_px[2] *= 0.2
    log_scale = np.log(s_px * z / cam["fx"]).astype(np.float32)
    quat = _unit_quats(rng, n)
    opacity = rng.normal(opacity_mu, opacity_sd, n).astype(np.float32)
    rgb = rng.uniform(0, 1, (3, n)).astype(np.float32)
    mask = np.where(rng.uniform(0, 1, n) < mask_keep, 3.0, -8.0).astype(np.float32)
    sc = SynthScene(mean, opacity, rgb, log_scale, quat, mask, dict(cam), [IDENTITY_VIEW.copy()])
    if codebook_LP:
        sc.codebook = random_codebooks(rng, log_scale, quat, *codebook_LP)
    return sc


def random_codebooks(rng, log_scale, quat, L, P, tie=None):
    """Seeded codebooks: stage 1 = P data vectors sampled without replacement
    (Fig 4 caption, read as R19); stage l >= 2 = zero-mean Gaussian
    residual codes whose spread shrinks by 0.35 per stage."""
    n = log_scale.shape[1]
    out = {}
    for name, x in (("scale_codes", log_scale), ("rot_codes", quat)):
        d = x.shape[0]
        codes = np.zeros((L, P, d), dtype=np.float32)
        pick = rng.choice(n, size=P, replace=n < P)
        codes[0] = x[:, pick].T
        spread = x.std(axis=1)
        for l in range(1, L):
            codes[l] = rng.normal(0, 1, (P, d)) * spread * (0.35 ** l)
        if tie is not None:
            a, b = tie
            codes[0, b] = codes[0, a]
        out[name] = codes
    return out


def replica_scene(seed=0, n=200_000):
    """C2: Replica-shaped 1200x680, 200k Gaussians, 75% kept masks, R-VQ 4x256."""
    return room_scene(n, CAMERAS["replica"], seed)


def tum_scene(seed=0, n=100_000):
    """C3: TUM-shaped 640x480, 100k Gaussians."""
    return room_scene(n, CAMERAS["tum"], seed)


def scannet_scene(seed=0, n=1_000_000, parity=False):
    """C4: ScanNet-shaped, 1M unpruned Gaussians, keep fraction 1/1.97."""
    sc = room_scene(n, CAMERAS["scannet"], seed, mask_keep=1.0 / 1.97)
    if parity:
        rng = np.random.default_rng(seed + 1000)
        sc.mask = rng.uniform(TAU_F32 - 2, TAU_F32 + 2, n).astype(np.float32)
    return sc


def look_view(centre, yaw):
    """World->camera [R|t] of a camera at `centre` looking along
    (cos yaw, 0, sin yaw) with image y along world +y."""
    f = np.array([math.cos(yaw), 0.0, math.sin(yaw)])
    y = np.array([0.0, 1.0, 0.0])
    x = np.cross(y, f)
    R = np.stack([x, y, f])
    t = -R @ np.asarray(centre, dtype=np.float64)
    return np.concatenate([R, t[:, None]], axis=1).astype(np.float32)


def window_scene(seed=0, n=500_000, n_keyframes=64, cam=None, codebook_LP=(4, 256)):
    """C5: Gaussians on the six faces of the box [-3,3]x[-1.5,1.5]x[-3,3]
    (area-weighted, 2 mm jitter) seen by n_keyframes inward-facing Replica
    cameras on a 1 m circle (yaw theta + pi + 0.3 sin 3 theta)."""
    rng = np.random.default_rng(seed)
    cam = dict(cam or CAMERAS["replica"])
    hx, hy, hz = 3.0, 1.5, 3.0
    faces = [  # (axis, sign, area)
        (0, -1, 4 * hy * hz), (0, 1, 4 * hy * hz), (1, -1, 4 * hx * hz), (1, 1, 4 * hx * hz),
        (2, -1, 4 * hx * hy), (2, 1, 4 * hx * hy)]
    areas = np.array([f[2] for f in faces])
    which = rng.choice(6, size=n, p=areas / areas.sum())
    pts = np.stack([rng.uniform(-hx, hx, n), rng.uniform(-hy, hy, n), rng.uniform(-hz, hz, n)])
    half = np.array([hx, hy, hz])
    for fi, (ax, sg, _) in enumerate(faces):
        sel = which == fi
        pts[ax, sel] = sg * half[ax]
    pts += rng.normal(0, 0.002, pts.shape)
    # distance to the camera circle (radius 1 m in the y = 0 plane)
    rxz = np.hypot(pts[0], pts[2])
    d = np.hypot(rxz - 1.0, pts[1])
    s_px = rng.lognormal(math.log(2.5), 0.35, (3, n))
    s_px[2] *= 0.2
    log_scale = np.log(s_px * np.maximum(d, 0.3) / cam["fx"]).astype(np.float32)
    quat = _unit_quats(rng, n)
    opacity = rng.normal(3.0, 1.5, n).astype(np.float32)
    rgb = rng.uniform(0, 1, (3, n)).astype(np.float32)
    mask = np.where(rng.uniform(0, 1, n) < 0.75, 3.0, -8.0).astype(np.float32)
    views = []
    for i in range(n_keyframes):
        th = 2 * math.pi * i / n_keyframes
        views.append(look_view((math.cos(th), 0.0, math.sin(th)), th + math.pi + 0.3 * math.sin(3 * th)))
    sc = SynthScene(pts.astype(np.float32), opacity, rgb, log_scale, quat, mask, cam, views)
    if codebook_LP:
        sc.codebook = random_codebooks(rng, log_scale, quat, *codebook_LP)
    return sc


def mid_scene(seed=0, n=3000, width=160, height=120):
    """Mid-size parity scene: several tiles in x and y plus a ragged tail
    (160x120 -> 10x8 tiles, the last tile row half empty)."""
    cam = dict(fx=0.5 * width * 1.25, fy=0.5 * width * 1.25, cx=width / 2 - 0.5,
               cy=height / 2 - 0.5, width=width, height=height, near=0.01, far=100.0)
    return room_scene(n, cam, seed, opacity_mu=0.5, codebook_LP=(2, 16))


def tiny_scene(seed=0, closed_form_centre=False):
    """C1: 64 Gaussians, 64x48 view, 2x16 R-VQ, adversarial masks and a depth tie."""
    rng = np.random.default_rng(seed)
    cam = dict(CAMERAS["tiny"])
    if closed_form_centre:
        cam["cx"], cam["cy"] = 32.0, 24.0
    n = 64
    W, H = cam["width"], cam["height"]
    px = rng.uniform(0, W - 1, n)
    py = rng.uniform(0, H - 1, n)
    z = rng.uniform(1, 3, n)
    # two Gaussians with a bit-identical depth inside one tile (tie test)
    px[1], py[1] = px[0] + 0.5, py[0] + 0.25
    z[1] = z[0]
    mean = np.stack([(px - cam["cx"]) / cam["fx"] * z, (py - cam["cy"]) / cam["fy"] * z, z])
    mean = mean.astype(np.float32)
    mean[2, 1] = mean[2, 0]
    s_px = rng.lognormal(math.log(2.5), 0.35, (3, n))
    s_px[2] *= 0.2
    log_scale = np.log(s_px * z / cam["fx"]).astype(np.float32)
    quat = _unit_quats(rng, n)
    opacity = rng.normal(0, 1.5, n).astype(np.float32)
    opacity[2] = 6.0     # alpha capped
    opacity[3] = -6.0    # culled by the 1/255 rule
    rgb = rng.uniform(0, 1, (3, n)).astype(np.float32)
    mask = np.full(n, 3.0, dtype=np.float32)
    perm = rng.permutation(np.arange(4, n))
    mask[perm[:12]] = -8.0
    mask[perm[12]] = TAU_F32                                  # exactly tau: masked
    mask[perm[13]] = np.nextafter(TAU_F32, np.float32(np.inf))  # just above: kept
    mask[perm[14]] = 0.0
    mask[perm[15]] = -0.0
    sc = SynthScene(mean, opacity, rgb, log_scale, quat, mask, cam, [IDENTITY_VIEW.copy()])
    sc.codebook = random_codebooks(rng, log_scale, quat, 2, 16, tie=(3, 15))
    return sc


def small_fd_scene(seed=0, n=20, width=32, height=32):
    """20-Gaussian 32x32 scene for finite-difference pins (smooth mode): all
    Gaussians in front of the camera and inside the image, o_hat < 1."""
    rng = np.random.default_rng(seed)
    cam = dict(fx=32.0, fy=32.0, cx=15.5, cy=15.5, width=width, height=height, near=0.01,
               far=100.0)
    px = rng.uniform(6, width - 7, n)
    py = rng.uniform(6, height - 7, n)
    # well-separated depths so a finite-difference step never reorders the list
    z = 1.5 + 1.5 * (rng.permutation(n) + rng.uniform(0.2, 0.8, n)) / n
    mean = np.stack([(px - cam["cx"]) / cam["fx"] * z, (py - cam["cy"]) / cam["fy"] * z, z])
    s_px = rng.lognormal(math.log(2.0), 0.3, (3, n))
    log_scale = np.log(s_px * z / cam["fx"])
    quat = _unit_quats(rng, n) * rng.uniform(0.7, 1.4, n)
    opacity = rng.normal(0, 1.0, n)
    rgb = rng.uniform(0, 1, (3, n))
    mask = rng.normal(1.0, 1.0, n)
    f = lambda a: np.asarray(a, dtype=np.float32)
    sc = SynthScene(f(mean), f(opacity), f(rgb), f(log_scale), f(quat), f(mask), cam,
                    [IDENTITY_VIEW.copy()])
    return sc


def perturbed_view(rng, rot_deg=2.0, trans=0.05):
    """A rigid world->camera view near identity (for pose tests / keyframes)."""
    axis = rng.standard_normal(3)
    axis /= np.linalg.norm(axis)
    th = math.radians(rot_deg)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    R = np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * (K @ K)
    t = rng.standard_normal(3) * trans
    return np.concatenate([R, t[:, None]], axis=1).astype(np.float32)


def upstream(rng, H, W):
    """Seeded N(0,1) upstream gradients dL/dC [3,H,W], dL/dD, dL/dS."""
    return (rng.standard_normal((3, H, W)).astype(np.float32),
            rng.standard_normal((H, W)).astype(np.float32),
            rng.standard_normal((H, W)).astype(np.float32))


def sample_patches(seed, n_keyframes, width, height, n_rays):
    """NEXT-4 ray sample (reading R30): n_rays // 64 distinct 8x8
    blocks drawn uniformly without replacement from all keyframes' whole
    blocks.  Returns one sorted int32 array of block ids (by * (W//8) + bx)
    per keyframe.  (The random draw of the method, passed in as an input.)"""
    bw, bh = width // 8, height // 8
    per = bw * bh
    n = min(n_rays // 64, n_keyframes * per)
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(n_keyframes * per, size=n, replace=False))
    kf = pick // per
    return [np.ascontiguousarray(pick[kf == k] % per, dtype=np.int32) for k in range(n_keyframes)]
