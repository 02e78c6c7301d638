"""CPU ORACLE for the csplat hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
(``paper_2403_11247_b200``) never imports it and shares no code with it.

This module is argument marshalling (numpy <-> ctypes) over ``liboracle.so``,
which is plain C11 built from ``oracle/*.c`` with ``-O2 -ffp-contract=off``.
Every function cites the PAPER.md passage it follows in the C source.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = ["oracle_project.c", "oracle_render.c", "oracle_rvq_prune.c", "oracle_loss.c"]

REC_WORDS = 16
TILE = 16


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, IEEE float32)."""
    srcs = [os.path.join(_HERE, s) for s in _SRCS]
    hdrs = [os.path.join(_HERE, h) for h in ("oracle.h", "oracle_internal.h")]
    if not force and os.path.exists(_SO):
        so_t = os.path.getmtime(_SO)
        if all(os.path.getmtime(s) <= so_t for s in srcs + hdrs):
            return _SO
    cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-fopenmp", "-Wall", "-o", _SO] + srcs + ["-lm"]
    subprocess.check_call(cmd)
    return _SO


class Camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32), ("near_z", C.c_float),
                ("far_z", C.c_float)]


class View(C.Structure):
    _fields_ = [("m", C.c_float * 12)]


class Params(C.Structure):
    _fields_ = [("mask_eps", C.c_float), ("alpha_max", C.c_float), ("t_min", C.c_float),
                ("dilation", C.c_float)]


class Gaussians(C.Structure):
    _fields_ = [("n", C.c_int64), ("mean", C.c_void_p), ("opacity", C.c_void_p),
                ("rgb", C.c_void_p), ("log_scale", C.c_void_p), ("quat", C.c_void_p),
                ("mask", C.c_void_p)]


class Codebook(C.Structure):
    _fields_ = [("stages", C.c_int32), ("size", C.c_int32), ("scale_codes", C.c_void_p),
                ("rot_codes", C.c_void_p), ("scale_idx", C.c_void_p), ("rot_idx", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_pexp.restype = C.c_float
        _lib.oracle_pexp.argtypes = [C.c_float]
        _lib.oracle_plog.restype = C.c_float
        _lib.oracle_plog.argtypes = [C.c_float]
        _lib.oracle_mask_tau.restype = C.c_float
        _lib.oracle_mask_tau.argtypes = [C.c_float]
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


@dataclass
class Scene:
    """Host-side scene in the ABI layout (planar SoA, float32)."""
    mean: np.ndarray       # [3, n]
    opacity: np.ndarray    # [n]
    rgb: np.ndarray        # [3, n]
    log_scale: np.ndarray  # [3, n]
    quat: np.ndarray       # [4, n]
    mask: np.ndarray       # [n]

    @property
    def n(self):
        return int(self.opacity.shape[0])


def _gauss(s: Scene, keep):
    arrs = [_f32(s.mean), _f32(s.opacity), _f32(s.rgb), _f32(s.log_scale), _f32(s.quat),
            _f32(s.mask)]
    keep.extend(arrs)
    return Gaussians(s.n, *[_p(a) for a in arrs])


def _codebook(cb, keep):
    if cb is None:
        return None
    sc, rc = _f32(cb["scale_codes"]), _f32(cb["rot_codes"])
    si = np.ascontiguousarray(cb["scale_idx"], dtype=np.uint16)
    ri = np.ascontiguousarray(cb["rot_idx"], dtype=np.uint16)
    keep.extend([sc, rc, si, ri])
    L, P = sc.shape[0], sc.shape[1]
    return Codebook(L, P, _p(sc), _p(rc), _p(si), _p(ri))


def camera(cam: dict) -> Camera:
    return Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], cam["width"], cam["height"],
                  cam.get("near", 0.01), cam.get("far", 100.0))


def view(v) -> View:
    vv = View()
    for i, x in enumerate(np.asarray(v, dtype=np.float32).reshape(12)):
        vv.m[i] = float(x)
    return vv


def params(mask_eps=0.01, alpha_max=0.99, t_min=1e-4, dilation=0.3) -> Params:
    return Params(mask_eps, alpha_max, t_min, dilation)


def set_threads(n: int = 1):
    """OpenMP threads of the oracle's loops (timed CPU baseline only; default 1)."""
    lib().oracle_set_threads(C.c_int32(n))


def set_flag_window(t_rel: float = 1e-5, cap_abs: float = 1e-6):
    """Ambiguity window of the forward's pixel flags."""
    lib().oracle_set_flag_window(C.c_double(t_rel), C.c_double(cap_abs))


def set_row_window(row_lo: int = 0, row_hi: int = -1):
    """Restrict render_fwd/render_bwd to pixel rows [row_lo, row_hi) (timing samples)."""
    lib().oracle_set_row_window(C.c_int32(row_lo), C.c_int32(row_hi))


def pexp(x: float) -> float:
    return lib().oracle_pexp(x)


def plog(x: float) -> float:
    return lib().oracle_plog(x)


def mask_tau(eps: float) -> float:
    return lib().oracle_mask_tau(eps)


def project(scene: Scene, cam: dict, v, prm: Params | None = None, codebook=None):
    """a3 (+a1, a2-decode): DA record [n,16] u32 and tile count [n] i32."""
    keep = []
    g = _gauss(scene, keep)
    cb = _codebook(codebook, keep)
    rec = np.zeros((scene.n, REC_WORDS), dtype=np.uint32)
    cnt = np.zeros(scene.n, dtype=np.int32)
    rc = lib().oracle_project(C.byref(g), C.byref(cb) if cb is not None else None,
                              C.byref(camera(cam)), C.byref(view(v)),
                              C.byref(prm or params()), _p(rec), _p(cnt))
    assert rc == 0, rc
    return rec, cnt


def tiles(cam: dict):
    tx = (cam["width"] + TILE - 1) // TILE
    ty = (cam["height"] + TILE - 1) // TILE
    return tx, ty


def bin_tiles(rec, cnt, cam: dict):
    """a4/a5: sorted pair gid list and per-tile [start, end)."""
    n = rec.shape[0]
    total = int(cnt.astype(np.int64).sum())
    tx, ty = tiles(cam)
    gid = np.zeros(max(total, 1), dtype=np.uint32)
    rng = np.zeros((tx * ty, 2), dtype=np.uint32)
    npairs = C.c_int64(0)
    rc = lib().oracle_bin_tiles(_p(np.ascontiguousarray(rec)), _p(np.ascontiguousarray(cnt)),
                                C.c_int64(n), C.byref(camera(cam)), C.c_int64(total), _p(gid),
                                _p(rng), C.byref(npairs))
    assert rc == 0, rc
    return gid[:total], rng


def render_fwd(rec, gid, rng, cam: dict, prm: Params | None = None):
    """a6: colour [3,H,W], depth, silhouette, T_final [H,W] (float64), n_contrib, flags, counters."""
    W, H = cam["width"], cam["height"]
    color = np.zeros((3, H, W)); depth = np.zeros((H, W)); sil = np.zeros((H, W))
    tfin = np.zeros((H, W)); ncon = np.zeros((H, W), dtype=np.int32)
    flags = np.zeros((H, W), dtype=np.uint8); counters = np.zeros(2, dtype=np.int64)
    gid = np.ascontiguousarray(gid, dtype=np.uint32)
    if gid.size == 0:
        gid = np.zeros(1, dtype=np.uint32)
    rc = lib().oracle_render_fwd(_p(np.ascontiguousarray(rec)), _p(gid),
                                 _p(np.ascontiguousarray(rng)), C.byref(camera(cam)),
                                 C.byref(prm or params()), _p(color), _p(depth), _p(sil), _p(tfin),
                                 _p(ncon), _p(flags), _p(counters))
    assert rc == 0
    return dict(color=color, depth=depth, sil=sil, t_final=tfin, n_contrib=ncon, flags=flags,
                e_pix=int(counters[0]), e_contrib=int(counters[1]))


def render_pixel(rec, cnt, cam: dict, px: int, py: int, prm: Params | None = None):
    """Untiled per-pixel definition: returns (C r, g, b, D, S, T), n composited."""
    out = np.zeros(6)
    ncomp = C.c_int32(0)
    rc = lib().oracle_render_pixel(_p(np.ascontiguousarray(rec)), _p(np.ascontiguousarray(cnt)),
                                   C.c_int64(rec.shape[0]), C.byref(camera(cam)),
                                   C.byref(prm or params()), C.c_int32(px), C.c_int32(py),
                                   _p(out), C.byref(ncomp))
    assert rc == 0
    return out, int(ncomp.value)


GRAD_NAMES = ["mean", "opacity", "rgb", "log_scale", "quat", "mask"]
GRAD_SLICES = {"mean": slice(0, 3), "opacity": slice(3, 4), "rgb": slice(4, 7),
               "log_scale": slice(7, 10), "quat": slice(10, 14), "mask": slice(14, 15)}


def render_bwd(scene: Scene, cam: dict, v, rec, gid, rng, d_color, d_depth, d_sil,
               prm: Params | None = None, codebook=None, zero_pixels=None, want_acc=False):
    """a7+a8: grads [15, n] float64, pose [6] (omega, v)."""
    keep = []
    g = _gauss(scene, keep)
    cb = _codebook(codebook, keep)
    n = scene.n
    grads = np.zeros((15, n)); pose = np.zeros(6)
    acc = np.zeros((n, 10)) if want_acc else None
    dC = np.ascontiguousarray(d_color, dtype=np.float64)
    dD = np.ascontiguousarray(d_depth, dtype=np.float64)
    dS = np.ascontiguousarray(d_sil, dtype=np.float64)
    zp = np.ascontiguousarray(zero_pixels, dtype=np.uint8) if zero_pixels is not None else None
    gid = np.ascontiguousarray(gid, dtype=np.uint32)
    if gid.size == 0:
        gid = np.zeros(1, dtype=np.uint32)
    rc = lib().oracle_render_bwd(C.byref(g), C.byref(cb) if cb is not None else None,
                                 C.byref(camera(cam)), C.byref(view(v)), C.byref(prm or params()),
                                 _p(np.ascontiguousarray(rec)), _p(gid),
                                 _p(np.ascontiguousarray(rng)), _p(dC), _p(dD), _p(dS), _p(zp),
                                 _p(grads), _p(pose), _p(acc))
    assert rc == 0
    out = {k: grads[s] for k, s in GRAD_SLICES.items()}
    out["pose"] = pose
    if want_acc:
        out["acc2d"] = acc
    return out


def smooth_render(scene: Scene, cam: dict, v, xi=None, prm: Params | None = None, clamp=False):
    keep = []
    g = _gauss(scene, keep)
    W, H = cam["width"], cam["height"]
    color = np.zeros((3, H, W)); depth = np.zeros((H, W)); sil = np.zeros((H, W))
    xia = np.ascontiguousarray(xi, dtype=np.float64) if xi is not None else None
    rc = lib().oracle_smooth_render(C.byref(g), C.byref(camera(cam)), C.byref(view(v)), _p(xia),
                                    C.byref(prm or params()), C.c_int32(int(clamp)), _p(color),
                                    _p(depth), _p(sil))
    assert rc == 0
    return color, depth, sil


def smooth_bwd(scene: Scene, cam: dict, v, d_color, d_depth, d_sil, prm: Params | None = None,
               clamp=False):
    keep = []
    g = _gauss(scene, keep)
    n = scene.n
    grads = np.zeros((15, n)); pose = np.zeros(6)
    rc = lib().oracle_smooth_bwd(C.byref(g), C.byref(camera(cam)), C.byref(view(v)),
                                 C.byref(prm or params()), C.c_int32(int(clamp)),
                                 _p(np.ascontiguousarray(d_color, dtype=np.float64)),
                                 _p(np.ascontiguousarray(d_depth, dtype=np.float64)),
                                 _p(np.ascontiguousarray(d_sil, dtype=np.float64)), _p(grads),
                                 _p(pose))
    assert rc == 0
    out = {k: grads[s] for k, s in GRAD_SLICES.items()}
    out["pose"] = pose
    return out


def tracking_loss(color, depth, sil, obs_color, obs_depth, lambda_d=1.0, gate=0.99):
    """NEXT-1 (Eq 12 + Eq 14 gate): upstream grads (dC, dD, dS), (L_t, L_c, L_d), flags."""
    color = np.ascontiguousarray(color, dtype=np.float64)
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    sil = np.ascontiguousarray(sil, dtype=np.float64)
    oc = _f32(obs_color)
    od = _f32(obs_depth)
    H, W = depth.shape
    dC = np.zeros_like(color); dD = np.zeros_like(depth); dS = np.zeros_like(sil)
    loss = np.zeros(3); flags = np.zeros((H, W), dtype=np.uint8)
    rc = lib().oracle_tracking_loss(_p(color), _p(depth), _p(sil), _p(oc), _p(od), C.c_int32(W),
                                    C.c_int32(H), C.c_double(lambda_d), C.c_double(gate), _p(dC),
                                    _p(dD), _p(dS), _p(loss), _p(flags))
    assert rc == 0
    return (dC, dD, dS), loss, flags


def ba_patch_loss(color, depth, obs_color, obs_depth, patches, n_rays, n_valid, lambda_d=1.0,
                  lambda_s=0.2, c1=0.01 ** 2, c2=0.03 ** 2):
    """NEXT-4 (reading R30): one keyframe's share of the patch BA loss.
    Returns (dC, dD, dS) upstream gradients and loss3 = its parts of
    (L_c, L_d, mean SSIM); L_ba = L_c + lambda_d L_d + lambda_s (1 - SSIM)."""
    color = np.ascontiguousarray(color, dtype=np.float64)
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    oc = _f32(obs_color)
    od = _f32(obs_depth)
    pt = np.ascontiguousarray(patches, dtype=np.int32)
    H, W = depth.shape
    dC = np.zeros_like(color); dD = np.zeros_like(depth); dS = np.zeros_like(depth)
    loss = np.zeros(3)
    rc = lib().oracle_ba_patch_loss(_p(color), _p(depth), _p(oc), _p(od), C.c_int32(W),
                                    C.c_int32(H), _p(pt), C.c_int64(pt.shape[0]),
                                    C.c_int64(n_rays), C.c_int64(n_valid), C.c_double(lambda_d),
                                    C.c_double(lambda_s), C.c_double(c1), C.c_double(c2),
                                    _p(dC), _p(dD), _p(dS), _p(loss))
    assert rc == 0
    return (dC, dD, dS), loss


def ba_count_valid(obs_depths, patches_per_kf, width):
    """|R| of Eq 12 over the sampled rays: patch pixels with a valid observed depth."""
    bw = width // 8
    n = 0
    for od, pt in zip(obs_depths, patches_per_kf):
        od = np.asarray(od, dtype=np.float32)
        for b in np.asarray(pt).ravel():
            by, bx = divmod(int(b), bw)
            n += int((od[8 * by:8 * by + 8, 8 * bx:8 * bx + 8] > 0).sum())
    return n


def mask_loss(mask, active, lam=1.0):
    """NEXT-3: Eq 8 over the active (in-frustum) Gaussians -> (L_m, d_mask)."""
    mask = _f32(mask)
    act = np.ascontiguousarray(active, dtype=np.uint8)
    d = np.zeros(mask.shape[0])
    lib().oracle_mask_loss.restype = C.c_double
    L = lib().oracle_mask_loss(_p(mask), _p(act), C.c_int64(mask.shape[0]), C.c_double(lam),
                               _p(d))
    return L, d


def keyframe_overlap(depth, cam: dict, cur_view, views):
    """NEXT-3: points of the current depth map inside each keyframe's frustum."""
    depth = _f32(depth)
    K = len(views)
    arr = (View * max(K, 1))(*[view(v) for v in views])
    counts = np.zeros(max(K, 1), dtype=np.int64)
    rc = lib().oracle_keyframe_overlap(_p(depth), C.byref(camera(cam)), C.byref(view(cur_view)),
                                       arr, C.c_int32(K), _p(counts))
    assert rc == 0
    return counts[:K]


def rvq_assign(x, codes):
    """a2: x [d, n] float32, codes [L, P, d] -> idx [L, n] u16, recon [d, n]."""
    x = _f32(x)
    codes = _f32(codes)
    d, n = x.shape
    L, P, d2 = codes.shape
    assert d2 == d
    idx = np.zeros((L, n), dtype=np.uint16)
    recon = np.zeros((d, n), dtype=np.float32)
    rc = lib().oracle_rvq_assign(_p(x), C.c_int64(n), C.c_int32(d), _p(codes), C.c_int32(L),
                                 C.c_int32(P), _p(idx), _p(recon))
    assert rc == 0
    return idx, recon


def rvq_code_grad(d_shat, idx, L, P, d_codes=None):
    """NEXT-2 STE: dL/dC^l[k] = sum of dL/dS_hat_n over i_n^l = k -> [L, P, d] float64."""
    g = np.ascontiguousarray(d_shat, dtype=np.float64)
    d, n = g.shape
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    acc = d_codes is not None
    out = np.ascontiguousarray(d_codes, dtype=np.float64) if acc else np.zeros((L, P, d))
    rc = lib().oracle_rvq_code_grad(_p(g), C.c_int64(n), C.c_int32(d), _p(idx), C.c_int32(L),
                                    C.c_int32(P), _p(out), C.c_int32(1 if acc else 0))
    assert rc == 0
    return out


def rvq_init_stage(x, codes, l, idx, sample):
    """NEXT-2 Fig 4: stage l of codes [L, P, d] := the stage-l residuals of x[:, sample]."""
    x = _f32(x)
    d, n = x.shape
    codes = np.array(codes, dtype=np.float32, copy=True)
    L, P = codes.shape[:2]
    idx = np.ascontiguousarray(idx, dtype=np.uint16) if idx is not None else \
        np.zeros((L, n), np.uint16)
    sample = np.ascontiguousarray(sample, dtype=np.int64)
    assert sample.shape == (P,)
    rc = lib().oracle_rvq_init_stage(_p(x), C.c_int64(n), C.c_int32(d), _p(codes), C.c_int32(L),
                                     C.c_int32(P), C.c_int32(l), _p(idx), _p(sample))
    assert rc == 0
    return codes


def rvq_update(x, codes, idx):
    """NEXT-2: k-means M-step for a given assignment -> (new codes, counts, losses[L+1])."""
    x = _f32(x)
    codes = _f32(codes)
    idx = np.ascontiguousarray(idx, dtype=np.uint16)
    d, n = x.shape
    L, P, _ = codes.shape
    out = np.zeros_like(codes)
    counts = np.zeros((L, P), dtype=np.int32)
    loss = np.zeros(L + 1)
    rc = lib().oracle_rvq_update(_p(x), C.c_int64(n), C.c_int32(d), _p(codes), C.c_int32(L),
                                 C.c_int32(P), _p(idx), _p(out), _p(counts), _p(loss))
    assert rc == 0
    return out, counts, loss


def mask_prune(planes: list, idx_planes: list, mask_plane: int, mask_eps=0.01,
               reset_mask=float("nan")):
    """a9: planes: list of float32 [n] arrays (one of them the mask logit)."""
    n = planes[0].shape[0]
    ins = [_f32(p) for p in planes]
    outs = [np.zeros(n, dtype=np.float32) for _ in planes]
    iins = [np.ascontiguousarray(p, dtype=np.uint16) for p in idx_planes]
    iouts = [np.zeros(n, dtype=np.uint16) for _ in idx_planes]
    PF = C.c_void_p * max(len(ins), 1)
    PI = C.c_void_p * max(len(iins), 1)
    keep_map = np.zeros(n, dtype=np.int32)
    nk = C.c_int64(0)
    rc = lib().oracle_mask_prune(C.c_int64(n), _p(ins[mask_plane]), C.c_float(mask_eps),
                                 C.c_int32(len(ins)), PF(*[a.ctypes.data for a in ins]),
                                 PF(*[a.ctypes.data for a in outs]), C.c_int32(len(iins)),
                                 PI(*[a.ctypes.data for a in iins]) if iins else None,
                                 PI(*[a.ctypes.data for a in iouts]) if iouts else None,
                                 C.c_int32(mask_plane), C.c_float(reset_mask), _p(keep_map),
                                 C.byref(nk))
    assert rc == 0
    k = int(nk.value)
    return [o[:k] for o in outs], [o[:k] for o in iouts], keep_map, k
