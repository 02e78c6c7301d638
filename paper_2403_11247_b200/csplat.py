"""Thin Python binding over libcsplat.so (include/csplat.h).

Argument marshalling only: torch tensors supply device memory and the current
CUDA stream; every step of the hot path runs in the library's sm_100a kernels.
There is no CPU fallback -- if the library is missing or the device is not a
B200 the calls raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSPLAT_LIB", os.path.join(_PKG, "libcsplat.so"))

TILE = 16
RECORD_BYTES = 64
SYNC, POSE_ONLY, ACCUMULATE, SKIP_CHAIN, WS_ZEROED = 1, 2, 4, 8, 16
PAIR_GID_MASK, PAIR_MASK_SHIFT = (1 << 28) - 1, 28  # pair_gid: index | block mask << 28
STATUS_CAPACITY, STATUS_CODE_INDEX = 1, 2  # device status bits (csplat.h)
OP_BIN_TILES, OP_RENDER_BWD, OP_MASK_PRUNE = 1, 2, 3


class CsplatError(RuntimeError):
    pass


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
    _fields_ = [("n", C.c_int64), ("n_dev", C.c_void_p), ("mean", C.c_void_p),
                ("opacity", C.c_void_p), ("rgb", C.c_void_p), ("log_scale", C.c_void_p),
                ("quat", C.c_void_p), ("mask", C.c_void_p)]


class GaussiansOut(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("mean", C.c_void_p), ("opacity", C.c_void_p),
                ("rgb", C.c_void_p), ("log_scale", C.c_void_p), ("quat", C.c_void_p),
                ("mask", C.c_void_p)]


class Codebook(C.Structure):
    _fields_ = [("stages", C.c_int32), ("size", C.c_int32), ("idx_bytes", C.c_int32),
                ("reserved", C.c_int32), ("scale_codes", C.c_void_p), ("rot_codes", C.c_void_p),
                ("scale_idx", C.c_void_p), ("rot_idx", C.c_void_p), ("status", C.c_void_p)]


class Grads(C.Structure):
    _fields_ = [("mean", C.c_void_p), ("opacity", C.c_void_p), ("rgb", C.c_void_p),
                ("log_scale", C.c_void_p), ("quat", C.c_void_p), ("mask", C.c_void_p),
                ("pose", C.c_void_p)]


EXPORTS = ["csplat_project", "csplat_bin_tiles", "csplat_render_fwd", "csplat_render_bwd",
           "csplat_rvq_assign", "csplat_mask_prune", "csplat_tracking_loss", "csplat_rvq_update",
           "csplat_mask_loss", "csplat_keyframe_overlap", "csplat_bin_tiles_active",
           "csplat_ba_patches", "csplat_ba_patch_loss", "csplat_project_dv",
           "csplat_render_bwd_dv", "csplat_pose_step", "csplat_tracking_bwd",
           "csplat_count_valid_depth",
           "csplat_workspace_bytes", "csplat_last_error", "csplat_status_string",
           "csplat_version"]
OP_TRACKING_LOSS = 4
OP_RVQ_UPDATE = 5
OP_MASK_LOSS = 6
OP_KEYFRAME_OVERLAP = 7

_lib = None


def lib():
    """Load libcsplat.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CsplatError(f"{LIB_PATH} is missing: build it with __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, u32 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32
        L.csplat_project.argtypes = [vp] * 8
        L.csplat_bin_tiles.argtypes = [vp, vp, i64, vp, i64, vp, vp, vp, u32, vp, C.c_size_t, vp]
        L.csplat_bin_tiles_active.argtypes = [vp, vp, i64, vp, vp, i64, vp, vp, vp, u32, vp,
                                              C.c_size_t, vp]
        L.csplat_ba_patches.argtypes = [vp, vp, vp, i64, vp, vp, vp]
        L.csplat_ba_patch_loss.argtypes = [vp] * 6 + [i64, i64, vp, C.c_float, C.c_float] + \
            [vp] * 5
        L.csplat_project_dv.argtypes = [vp] * 8
        L.csplat_project_bin.argtypes = [vp] * 8 + [i64, vp, vp, vp, u32, vp, C.c_size_t, vp]
        L.csplat_project_bin_render.argtypes = [vp] * 7 + [i64, vp, vp, vp, vp, C.c_size_t] + \
            [vp] * 6
        L.csplat_project_bin_render_dv.argtypes = L.csplat_project_bin_render.argtypes
        L.csplat_render_step.argtypes = [vp] * 7 + [i64, vp, vp, vp, vp, C.c_size_t] + \
            [vp] * 8 + [u32, vp, vp, C.c_size_t, vp]
        L.csplat_tracking_step.argtypes = [vp] * 8 + [i64, vp, vp, vp, vp, C.c_size_t] + \
            [vp] * 8 + [C.c_float, C.c_float, u32, vp, vp, vp, C.c_size_t, vp]
        L.csplat_project_bin_dv.argtypes = [vp] * 8 + [i64, vp, vp, vp, u32, vp, C.c_size_t,
                                                        vp]
        L.csplat_render_bwd_dv.argtypes = [vp] * 13 + [u32, vp, vp, C.c_size_t, vp]
        L.csplat_pose_step.argtypes = [vp, vp, C.c_float, C.c_float, vp]
        L.csplat_tracking_bwd.argtypes = [vp] * 17 + [C.c_float, C.c_float, u32, vp, vp, vp,
                                                      C.c_size_t, vp]
        L.csplat_count_valid_depth.argtypes = [vp, i32, i32, vp, vp]
        L.csplat_render_fwd.argtypes = [vp] * 11
        L.csplat_render_bwd.argtypes = [vp] * 13 + [u32, vp, vp, C.c_size_t, vp]
        L.csplat_rvq_assign.argtypes = [vp, i64, vp, i32, vp, i32, i32, vp, i32, vp, vp]
        L.csplat_project_views.argtypes = [vp] * 4 + [i32, vp, vp, vp, vp]
        L.csplat_project_bin_views.argtypes = [vp] * 4 + [i32] + [vp] * 3 + [i64, i32] + \
            [vp] * 2 + [i64] + [vp] * 4 + [C.c_size_t, vp]
        L.csplat_render_fwd_list.argtypes = [vp] * 4 + [i32] + [vp] * 8
        L.csplat_render_bwd_list.argtypes = [vp] * 9 + [i32] + [vp] * 5 + [u32, vp, vp,
                                                                       C.c_size_t, vp]
        L.csplat_chain_views.argtypes = [vp] * 4 + [i32, vp, vp, vp, u32, vp, vp]
        L.csplat_rvq_code_grad.argtypes = [vp, i64, vp, i32, vp, i32, i32, i32, vp, u32, vp]
        L.csplat_rvq_init_stage.argtypes = [vp, i64, i32, vp, i32, i32, i32, vp, i32, vp, vp]
        L.csplat_mask_prune.argtypes = [vp, vp, C.c_float, C.c_float, vp, vp, vp, vp, vp, vp,
                                        C.c_size_t, vp]
        L.csplat_tracking_loss.argtypes = [vp] * 5 + [i32, i32, C.c_float, C.c_float] + \
            [vp] * 5 + [C.c_size_t, vp]
        L.csplat_rvq_update.argtypes = [vp, i64, vp, i32, vp, i32, i32, vp, i32, vp, vp, vp, vp,
                                        C.c_size_t, vp]
        L.csplat_mask_loss.argtypes = [vp, vp, C.c_float, vp, vp, vp, C.c_size_t, vp]
        L.csplat_keyframe_overlap.argtypes = [vp, vp, vp, vp, i32, vp, vp, C.c_size_t, vp]
        L.csplat_workspace_bytes.argtypes = [C.c_int, i64, i64, vp]
        L.csplat_workspace_bytes.restype = C.c_size_t
        L.csplat_last_error.argtypes = [C.c_char_p, C.c_size_t]
        L.csplat_status_string.argtypes = [C.c_int]
        L.csplat_status_string.restype = C.c_char_p
        for name in EXPORTS:
            if name not in ("csplat_workspace_bytes", "csplat_status_string"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        buf = C.create_string_buffer(512)
        lib().csplat_last_error(buf, 512)
        raise CsplatError(f"{what}: {lib().csplat_status_string(status).decode()} "
                          f"({buf.value.decode(errors='replace')})")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def camera(cam: dict) -> Camera:
    return Camera(cam["fx"], cam["fy"], cam["cx"], cam["cy"], cam["width"], cam["height"],
                  cam.get("near", 0.01), cam.get("far", 100.0))


def view(v) -> View:
    vv = View()
    vals = v.reshape(-1).tolist() if hasattr(v, "reshape") else list(v)
    for i, x in enumerate(vals[:12]):
        vv.m[i] = float(x)
    return vv


def params(mask_eps=0.01, alpha_max=0.99, t_min=1e-4, dilation=0.3) -> Params:
    return Params(mask_eps, alpha_max, t_min, dilation)


def tiles(cam: dict):
    return (cam["width"] + TILE - 1) // TILE, (cam["height"] + TILE - 1) // TILE


@dataclass
class GaussianMap:
    """Device SoA planes (float32, contiguous) in the ABI layout."""
    mean: torch.Tensor       # [3, n]
    opacity: torch.Tensor    # [n]
    rgb: torch.Tensor        # [3, n]
    log_scale: torch.Tensor  # [3, n]
    quat: torch.Tensor       # [4, n]
    mask: torch.Tensor       # [n]
    n_dev: torch.Tensor | None = None

    @property
    def n(self):
        return int(self.opacity.shape[-1])

    @staticmethod
    def from_numpy(planes: dict, device="cuda"):
        return GaussianMap(**{k: torch.as_tensor(planes[k], dtype=torch.float32).contiguous()
                              .to(device) for k in ("mean", "opacity", "rgb", "log_scale",
                                                    "quat", "mask")})

    def struct(self) -> Gaussians:
        return Gaussians(self.n, _ptr(self.n_dev), _ptr(self.mean), _ptr(self.opacity),
                         _ptr(self.rgb), _ptr(self.log_scale), _ptr(self.quat), _ptr(self.mask))


@dataclass
class CodebookT:
    scale_codes: torch.Tensor  # [L, P, 3]
    rot_codes: torch.Tensor    # [L, P, 4]
    scale_idx: torch.Tensor    # [L, n] uint8/int16
    rot_idx: torch.Tensor
    status: torch.Tensor | None = None  # [1] int32 device status word (STATUS_CODE_INDEX)

    def struct(self) -> Codebook:
        L, P = self.scale_codes.shape[:2]
        ib = self.scale_idx.element_size()
        return Codebook(L, P, ib, 0, _ptr(self.scale_codes), _ptr(self.rot_codes),
                        _ptr(self.scale_idx), _ptr(self.rot_idx), _ptr(self.status))


def release_thread_resources():
    """csplat_release_thread_resources: free this thread's fork streams / events."""
    _check(lib().csplat_release_thread_resources(), "csplat_release_thread_resources")


def alloc_tile_range(cam: dict, device) -> torch.Tensor:
    """tile_range [T + 1, 2] int32: the T tile ranges plus the view's status slot
    {status word, max n_pairs} (csplat.h), zeroed here; the library only ORs /
    maxes into the slot, so it collects every call until the caller clears it."""
    tx, ty = tiles(cam)
    return torch.zeros((tx * ty + 1, 2), dtype=torch.int32, device=device)


def range_status(tile_range: torch.Tensor) -> torch.Tensor:
    """The status slot of tile_range (device tensor [2]: status bits, max n_pairs)."""
    return tile_range[-1]


def clear_status(tile_range: torch.Tensor):
    tile_range[-1].zero_()


def _byref(x):
    return C.byref(x) if x is not None else None


def project(g: GaussianMap, cam: dict, v, prm: Params | None = None, cb: CodebookT | None = None,
            rec=None, count=None, stream=None):
    """a1+a2(decode)+a3.  Returns (rec [n,16] int32 view of the 64-B records, count [n])."""
    n = g.n
    dev = g.opacity.device
    rec = rec if rec is not None else torch.empty((max(n, 1), 16), dtype=torch.int32, device=dev)
    count = count if count is not None else torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    if _on_device(v):  # the view is read by the kernel (graph-captured pose updates)
        _check(lib().csplat_project_dv(C.byref(gs), _byref(cbs), C.byref(camera(cam)), _ptr(v),
                                       C.byref(prm or params()), _ptr(rec), _ptr(count),
                                       _stream(stream)), "csplat_project_dv")
        return rec[:n], count[:n]
    _check(lib().csplat_project(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                C.byref(view(v)), C.byref(prm or params()), _ptr(rec),
                                _ptr(count), _stream(stream)), "csplat_project")
    return rec[:n], count[:n]


def project_bin(g: GaussianMap, cam: dict, v, capacity: int, prm: Params | None = None,
                cb: CodebookT | None = None, rec=None, count=None, ws=None, out=None, sync=True,
                stream=None, tile_active=None):
    """a1+a2(decode)+a3+a4+a5 in one call (the bucket pass fused into the projection):
    the outputs of project() and bin_tiles().  Returns (rec, count, bin dict)."""
    n = g.n
    dev = g.opacity.device
    rec = rec if rec is not None else torch.empty((max(n, 1), 16), dtype=torch.int32, device=dev)
    count = count if count is not None else torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    tx, ty = tiles(cam)
    if out is None:
        out = dict(pair_gid=torch.empty(max(capacity, 1), dtype=torch.int32, device=dev),
                   tile_range=alloc_tile_range(cam, dev),
                   n_pairs_dev=torch.zeros(1, dtype=torch.int64, device=dev))
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_BIN_TILES, n, capacity, cam), dtype=torch.uint8,
                         device=dev)
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    tail = (_ptr(tile_active), capacity, _ptr(out["pair_gid"]),
            _ptr(out["tile_range"]), _ptr(out["n_pairs_dev"]), SYNC if sync else 0, _ptr(ws),
            ws.numel(), _stream(stream))
    if _on_device(v):
        _check(lib().csplat_project_bin_dv(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                           _ptr(v), C.byref(prm or params()), _ptr(rec),
                                           _ptr(count), *tail), "csplat_project_bin_dv")
    else:
        _check(lib().csplat_project_bin(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                        C.byref(view(v)), C.byref(prm or params()), _ptr(rec),
                                        _ptr(count), *tail), "csplat_project_bin")
    return rec[:n], count[:n], out


def project_bin_render(g: GaussianMap, cam: dict, v, capacity: int, prm: Params | None = None,
                       cb: CodebookT | None = None, rec=None, count=None, ws=None, out=None,
                       img=None, stream=None):
    """project_bin + render_fwd in one call (the sort and the forward pipelined in
    tile chunks on two library streams).  Returns (rec, count, bin dict, img dict)."""
    n = g.n
    dev = g.opacity.device
    H, W = cam["height"], cam["width"]
    rec = rec if rec is not None else torch.empty((max(n, 1), 16), dtype=torch.int32, device=dev)
    count = count if count is not None else torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    tx, ty = tiles(cam)
    if out is None:
        out = dict(pair_gid=torch.empty(max(capacity, 1), dtype=torch.int32, device=dev),
                   tile_range=alloc_tile_range(cam, dev),
                   n_pairs_dev=torch.zeros(1, dtype=torch.int64, device=dev))
    if img is None:
        img = dict(color=torch.empty((3, H, W), device=dev), depth=torch.empty((H, W), device=dev),
                   sil=torch.empty((H, W), device=dev), t_final=torch.empty((H, W), device=dev),
                   n_contrib=torch.empty((H, W), dtype=torch.int32, device=dev))
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_BIN_TILES, n, capacity, cam), dtype=torch.uint8,
                         device=dev)
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    tail = (_ptr(rec), _ptr(count), capacity, _ptr(out["pair_gid"]),
            _ptr(out["tile_range"]), _ptr(out["n_pairs_dev"]), _ptr(ws), ws.numel(),
            _ptr(img["color"]), _ptr(img["depth"]), _ptr(img["sil"]), _ptr(img["t_final"]),
            _ptr(img["n_contrib"]), _stream(stream))
    if _on_device(v):
        _check(lib().csplat_project_bin_render_dv(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                                  _ptr(v), C.byref(prm or params()), *tail),
               "csplat_project_bin_render_dv")
    else:
        _check(lib().csplat_project_bin_render(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                               C.byref(view(v)), C.byref(prm or params()), *tail),
               "csplat_project_bin_render")
    return rec[:n], count[:n], out, img


def render_step(g: GaussianMap, cam: dict, v, capacity: int, d_color, d_depth, d_sil,
                prm: Params | None = None, cb: CodebookT | None = None, flags: int = 0,
                rec=None, count=None, ws=None, out=None, img=None, grads=None, ws_bwd=None,
                stream=None):
    """a3 .. a8 for one view in one call (csplat_render_step: per tile chunk the
    sort, the forward and the backward kernel on a library stream, then the
    chain).  Returns (rec, count, bin dict, img dict, grads dict)."""
    n = g.n
    dev = g.opacity.device
    H, W = cam["height"], cam["width"]
    rec = rec if rec is not None else torch.empty((max(n, 1), 16), dtype=torch.int32, device=dev)
    count = count if count is not None else torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    tx, ty = tiles(cam)
    if out is None:
        out = dict(pair_gid=torch.empty(max(capacity, 1), dtype=torch.int32, device=dev),
                   tile_range=alloc_tile_range(cam, dev),
                   n_pairs_dev=torch.zeros(1, dtype=torch.int64, device=dev))
    if img is None:
        img = dict(color=torch.empty((3, H, W), device=dev), depth=torch.empty((H, W), device=dev),
                   sil=torch.empty((H, W), device=dev), t_final=torch.empty((H, W), device=dev),
                   n_contrib=torch.empty((H, W), dtype=torch.int32, device=dev))
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_BIN_TILES, n, capacity, cam), dtype=torch.uint8,
                         device=dev)
    if grads is None:
        grads = alloc_grads(n, dev)
    if ws_bwd is None:
        ws_bwd = torch.empty(workspace_bytes(OP_RENDER_BWD, n), dtype=torch.uint8, device=dev)
    gr = Grads(*[_ptr(grads.get(k)) for k in ("mean", "opacity", "rgb", "log_scale", "quat",
                                               "mask", "pose")])
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    _check(lib().csplat_render_step(
        C.byref(gs), _byref(cbs), C.byref(camera(cam)), C.byref(view(v)),
        C.byref(prm or params()), _ptr(rec), _ptr(count), capacity, _ptr(out["pair_gid"]),
        _ptr(out["tile_range"]), _ptr(out["n_pairs_dev"]), _ptr(ws),
        ws.numel(), _ptr(img["color"]), _ptr(img["depth"]), _ptr(img["sil"]),
        _ptr(img["t_final"]), _ptr(img["n_contrib"]), _ptr(d_color), _ptr(d_depth), _ptr(d_sil),
        flags, C.byref(gr), _ptr(ws_bwd), ws_bwd.numel(), _stream(stream)), "csplat_render_step")
    return rec[:n], count[:n], out, img, grads


def tracking_step(g: GaussianMap, cam: dict, v, capacity: int, obs_color, obs_depth, n_valid,
                  prm: Params | None = None, cb: CodebookT | None = None,
                  flags: int = POSE_ONLY, lambda_depth=1.0, sil_gate=0.99, rec=None, count=None,
                  ws=None, out=None, img=None, grads=None, loss3=None, ws_bwd=None, stream=None):
    """NEXT-1: one tracking iteration's render in one call (csplat_tracking_step):
    project + bin + fwd + the loss-fused backward per tile chunk, then the chain.
    Returns (grads, loss3)."""
    n = g.n
    dev = g.opacity.device
    if grads is None:
        grads = alloc_grads(n, dev, pose_only=bool(flags & POSE_ONLY))
    if loss3 is None:
        loss3 = torch.zeros(3, device=dev)
    if ws_bwd is None:
        ws_bwd = torch.empty(workspace_bytes(OP_RENDER_BWD, n), dtype=torch.uint8, device=dev)
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_BIN_TILES, n, capacity, cam), dtype=torch.uint8,
                         device=dev)
    gr = Grads(*[_ptr(grads.get(k)) for k in ("mean", "opacity", "rgb", "log_scale", "quat",
                                               "mask", "pose")])
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    dv = _on_device(v)
    hv = None if dv else view(v)
    _check(lib().csplat_tracking_step(
        C.byref(gs), _byref(cbs), C.byref(camera(cam)), None if dv else C.byref(hv),
        _ptr(v) if dv else None, C.byref(prm or params()), _ptr(rec), _ptr(count), capacity,
        _ptr(out["pair_gid"]), _ptr(out["tile_range"]),
        _ptr(out["n_pairs_dev"]), _ptr(ws), ws.numel(), _ptr(img["color"]), _ptr(img["depth"]),
        _ptr(img["sil"]), _ptr(img["t_final"]), _ptr(img["n_contrib"]), _ptr(obs_color),
        _ptr(obs_depth), _ptr(n_valid), lambda_depth, sil_gate, flags, C.byref(gr), _ptr(loss3),
        _ptr(ws_bwd), ws_bwd.numel(), _stream(stream)), "csplat_tracking_step")
    return grads, loss3


def _on_device(v) -> bool:
    if isinstance(v, torch.Tensor) and v.is_cuda:
        if v.dtype != torch.float32 or v.numel() != 12 or not v.is_contiguous():
            raise CsplatError("a device view must be a contiguous float32 tensor of 12 values")
        return True
    return False


def count_valid_depth(obs_depth, n_valid=None, stream=None):
    """|R| of Eq 12: pixels of obs_depth [H, W] with a valid depth -> device int64[1]."""
    H, W = obs_depth.shape
    if n_valid is None:
        n_valid = torch.zeros(1, dtype=torch.int64, device=obs_depth.device)
    _check(lib().csplat_count_valid_depth(_ptr(obs_depth), W, H, _ptr(n_valid), _stream(stream)),
           "csplat_count_valid_depth")
    return n_valid


def tracking_bwd(g: GaussianMap, cam: dict, v, rec, pair_gid, tile_range, img: dict, obs_color,
                 obs_depth, n_valid, prm: Params | None = None, cb: CodebookT | None = None,
                 flags: int = POSE_ONLY, lambda_depth=1.0, sil_gate=0.99, grads=None, loss3=None,
                 ws=None, stream=None):
    """NEXT-1 loss-fused backward: render_bwd with the Eq 12 + Eq 14 upstream formed
    in the kernel from the rendered `img` (render_fwd output) and the observed frame."""
    n = g.n
    dev = g.opacity.device
    if grads is None:
        grads = alloc_grads(n, dev, pose_only=bool(flags & POSE_ONLY))
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_RENDER_BWD, n), dtype=torch.uint8, device=dev)
    gr = Grads(*[_ptr(grads.get(k)) for k in ("mean", "opacity", "rgb", "log_scale", "quat",
                                               "mask", "pose")])
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    dv = _on_device(v)
    hv = None if dv else view(v)
    _check(lib().csplat_tracking_bwd(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                     None if dv else C.byref(hv), _ptr(v) if dv else None,
                                     C.byref(prm or params()), _ptr(rec), _ptr(pair_gid),
                                     _ptr(tile_range), _ptr(img["t_final"]), _ptr(img["n_contrib"]),
                                     _ptr(img["color"]), _ptr(img["depth"]), _ptr(img["sil"]),
                                     _ptr(obs_color), _ptr(obs_depth), _ptr(n_valid),
                                     lambda_depth, sil_gate, flags, C.byref(gr), _ptr(loss3),
                                     _ptr(ws), ws.numel(), _stream(stream)),
           "csplat_tracking_bwd")
    return grads


def pose_step(view_dev, pose_grad, lr_rot: float, lr_trans: float, stream=None):
    """NEXT-1: view_dev <- Exp(-(lr_rot g_omega, lr_trans g_v)) view_dev on the device."""
    _on_device(view_dev)
    _check(lib().csplat_pose_step(_ptr(view_dev), _ptr(pose_grad), lr_rot, lr_trans,
                                  _stream(stream)), "csplat_pose_step")
    return view_dev


def workspace_bytes(op: int, n: int, pairs: int = 0, cam: dict | None = None) -> int:
    c = camera(cam) if cam is not None else None
    return int(lib().csplat_workspace_bytes(op, n, pairs, _byref(c)))


def bin_tiles(rec, count, cam: dict, capacity: int, ws=None, out=None, sync=True, stream=None,
              tile_active=None):
    """a4+a5.  Returns dict(pair_gid, tile_range, n_pairs_dev).
    tile_active (device int32 bitmask, NEXT-4): bin only those tiles."""
    n = int(count.shape[0])
    dev = rec.device
    tx, ty = tiles(cam)
    if out is None:
        out = dict(pair_gid=torch.empty(max(capacity, 1), dtype=torch.int32, device=dev),
                   tile_range=alloc_tile_range(cam, dev),
                   n_pairs_dev=torch.zeros(1, dtype=torch.int64, device=dev))
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_BIN_TILES, n, capacity, cam), dtype=torch.uint8,
                         device=dev)
    if tile_active is None:
        st = lib().csplat_bin_tiles(_ptr(rec), _ptr(count), n, C.byref(camera(cam)), capacity,
                                    _ptr(out["pair_gid"]),
                                    _ptr(out["tile_range"]), _ptr(out["n_pairs_dev"]),
                                    SYNC if sync else 0, _ptr(ws), ws.numel(), _stream(stream))
        _check(st, "csplat_bin_tiles")
    else:
        st = lib().csplat_bin_tiles_active(_ptr(rec), _ptr(count), n, C.byref(camera(cam)),
                                           _ptr(tile_active), capacity, _ptr(out["pair_gid"]),
                                           _ptr(out["tile_range"]),
                                           _ptr(out["n_pairs_dev"]), SYNC if sync else 0,
                                           _ptr(ws), ws.numel(), _stream(stream))
        _check(st, "csplat_bin_tiles_active")
    return out


def render_fwd(rec, pair_gid, tile_range, cam: dict, prm: Params | None = None, out=None,
               stream=None, tile_list=None, max_tiles: int = 0):
    """a6.  Returns dict(color [3,H,W], depth, sil, t_final [H,W], n_contrib [H,W])."""
    H, W = cam["height"], cam["width"]
    dev = tile_range.device
    if out is None:
        out = dict(color=torch.empty((3, H, W), device=dev),
                   depth=torch.empty((H, W), device=dev), sil=torch.empty((H, W), device=dev),
                   t_final=torch.empty((H, W), device=dev),
                   n_contrib=torch.empty((H, W), dtype=torch.int32, device=dev))
    if tile_list is not None:  # only the listed tiles ({count, tiles...})
        _check(lib().csplat_render_fwd_list(
            _ptr(rec), _ptr(pair_gid), _ptr(tile_range), _ptr(tile_list), int(max_tiles),
            C.byref(camera(cam)), C.byref(prm or params()), _ptr(out["color"]), _ptr(out["depth"]),
            _ptr(out["sil"]), _ptr(out["t_final"]), _ptr(out["n_contrib"]), _stream(stream)),
            "csplat_render_fwd_list")
        return out
    _check(lib().csplat_render_fwd(_ptr(rec), _ptr(pair_gid), _ptr(tile_range), C.byref(camera(cam)),
                                   C.byref(prm or params()), _ptr(out["color"]),
                                   _ptr(out["depth"]), _ptr(out["sil"]), _ptr(out["t_final"]),
                                   _ptr(out["n_contrib"]), _stream(stream)), "csplat_render_fwd")
    return out


GRAD_SHAPES = dict(mean=3, opacity=1, rgb=3, log_scale=3, quat=4, mask=1)


def _views_arr(views):
    arr = (View * max(len(views), 1))(*[view(v) for v in views])
    return arr


def project_views(g: GaussianMap, cam: dict, views, prm: Params | None = None,
                  cb: CodebookT | None = None, rec=None, count=None, stream=None):
    """a1-a3 over V views reading each Gaussian once: rec [V, n, 16], count [V, n]."""
    n, V = g.n, len(views)
    dev = g.opacity.device
    rec = rec if rec is not None else torch.empty((V, max(n, 1), 16), dtype=torch.int32, device=dev)
    count = count if count is not None else torch.empty((V, max(n, 1)), dtype=torch.int32,
                                                        device=dev)
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    _check(lib().csplat_project_views(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                      _views_arr(views), V, C.byref(prm or params()), _ptr(rec),
                                      _ptr(count), _stream(stream)), "csplat_project_views")
    return rec, count


def ws_bin_per_view(n: int, capacity: int, cam: dict) -> int:
    """csplat_project_bin_views' workspace bytes per view (a multiple of 256)."""
    b = workspace_bytes(OP_BIN_TILES, n, capacity, cam)
    return (b + 255) // 256 * 256


def alloc_views(n: int, V: int, capacity: int, cam: dict, device):
    """Per-view buffers of csplat_project_bin_views for V views."""
    tx, ty = tiles(cam)
    wsv = ws_bin_per_view(n, capacity, cam)
    return dict(rec=torch.empty((V, max(n, 1), 16), dtype=torch.int32, device=device),
                count=torch.empty((V, max(n, 1)), dtype=torch.int32, device=device),
                pair_gid=torch.empty((V, max(capacity, 1)), dtype=torch.int32, device=device),
                tile_range=torch.zeros((V, tx * ty + 1, 2), dtype=torch.int32, device=device),
                n_pairs_dev=torch.zeros(V, dtype=torch.int64, device=device),
                ws=torch.empty(V * wsv + 256, dtype=torch.uint8, device=device), ws_per_view=wsv,
                capacity=capacity)


def project_bin_views(g: GaussianMap, cam: dict, views, out: dict, prm: Params | None = None,
                      cb: CodebookT | None = None, tile_active=None, tile_lists=None,
                      max_list: int = 0, stream=None):
    """a1-a5 over V views (projection once per Gaussian + per-view bucket + one
    batched sort) into the per-view buffers of alloc_views."""
    V = len(views)
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    ws = out["ws"]
    base = ws.data_ptr()
    off = (-base) % 256                     # 256-byte aligned workspace base
    _check(lib().csplat_project_bin_views(
        C.byref(gs), _byref(cbs), C.byref(camera(cam)), _views_arr(views), V,
        C.byref(prm or params()), _ptr(tile_active), _ptr(tile_lists),
        int(tile_lists.shape[1]) if tile_lists is not None else 0, int(max_list),
        _ptr(out["rec"]), _ptr(out["count"]),
        out["capacity"], _ptr(out["pair_gid"]), _ptr(out["tile_range"]), _ptr(out["n_pairs_dev"]),
        C.c_void_p(base + off), out["ws_per_view"], _stream(stream)), "csplat_project_bin_views")
    return out


def chain_views(g: GaussianMap, cam: dict, views, rec, ws, grads: dict, pose=None,
                prm: Params | None = None, cb: CodebookT | None = None, flags: int = 0,
                stream=None):
    """a8 summed over V views: ws [V, OP_RENDER_BWD bytes] (render_bwd SKIP_CHAIN
    workspaces, 256-byte aligned), grads planes (overwritten unless ACCUMULATE),
    pose [V, 6] (optional)."""
    V = len(views)
    gr = Grads(*[_ptr(grads.get(k)) for k in ("mean", "opacity", "rgb", "log_scale", "quat",
                                               "mask")], _ptr(pose))
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    _check(lib().csplat_chain_views(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                    _views_arr(views), V, C.byref(prm or params()), _ptr(rec),
                                    _ptr(ws), flags, C.byref(gr), _stream(stream)),
           "csplat_chain_views")
    return grads


def alloc_grads(n: int, device="cuda", pose_only=False):
    """Gradient planes as views of ONE flat float32 buffer ``g["flat"]``
    ([15 n] planes then the 6 pose entries) so a data-parallel step can
    all-reduce them with a single collective."""
    total = (0 if pose_only else 15 * n) + 8
    flat = torch.zeros(total, device=device)
    g = {"flat": flat}
    off = 0
    if not pose_only:
        for k, c in GRAD_SHAPES.items():
            g[k] = flat[off:off + c * n].view((c, n) if c > 1 else (n,))
            off += c * n
    g["pose"] = flat[off:off + 6]
    return g


def render_bwd(g: GaussianMap, cam: dict, v, rec, pair_gid, tile_range, t_final, n_contrib,
               d_color, d_depth, d_sil, prm: Params | None = None, cb: CodebookT | None = None,
               flags: int = 0, grads=None, ws=None, stream=None, tile_list=None,
               max_tiles: int = 0):
    """a7+a8.  Returns the grads dict (mean, opacity, rgb, log_scale, quat, mask, pose)."""
    n = g.n
    dev = g.opacity.device
    if grads is None:
        grads = alloc_grads(n, dev, pose_only=bool(flags & POSE_ONLY))
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_RENDER_BWD, n), dtype=torch.uint8, device=dev)
    gr = Grads(*[_ptr(grads.get(k)) for k in ("mean", "opacity", "rgb", "log_scale", "quat",
                                               "mask", "pose")])
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    if tile_list is not None:  # only the listed tiles ({count, tiles...})
        _check(lib().csplat_render_bwd_list(
            C.byref(gs), _byref(cbs), C.byref(camera(cam)), C.byref(view(v)),
            C.byref(prm or params()), _ptr(rec), _ptr(pair_gid), _ptr(tile_range), _ptr(tile_list),
            int(max_tiles), _ptr(t_final), _ptr(n_contrib), _ptr(d_color), _ptr(d_depth),
            _ptr(d_sil), flags, C.byref(gr), _ptr(ws), ws.numel(), _stream(stream)),
            "csplat_render_bwd_list")
        return grads
    if _on_device(v):
        _check(lib().csplat_render_bwd_dv(C.byref(gs), _byref(cbs), C.byref(camera(cam)), _ptr(v),
                                          C.byref(prm or params()), _ptr(rec), _ptr(pair_gid),
                                          _ptr(tile_range), _ptr(t_final), _ptr(n_contrib),
                                          _ptr(d_color), _ptr(d_depth), _ptr(d_sil), flags,
                                          C.byref(gr), _ptr(ws), ws.numel(), _stream(stream)),
               "csplat_render_bwd_dv")
        return grads
    _check(lib().csplat_render_bwd(C.byref(gs), _byref(cbs), C.byref(camera(cam)),
                                   C.byref(view(v)), C.byref(prm or params()), _ptr(rec),
                                   _ptr(pair_gid), _ptr(tile_range), _ptr(t_final),
                                   _ptr(n_contrib), _ptr(d_color), _ptr(d_depth), _ptr(d_sil),
                                   flags, C.byref(gr), _ptr(ws), ws.numel(), _stream(stream)),
           "csplat_render_bwd")
    return grads


def tracking_loss(img: dict, obs_color, obs_depth, lambda_depth=1.0, sil_gate=0.99, out=None,
                  loss3=None, ws=None, stream=None):
    """NEXT-1 (Eq 12 gated by Eq 14): upstream grads (d_color, d_depth, d_sil) of the
    rendered images `img` (render_fwd output) and loss3 = (L_t, L_c, L_d) on the device."""
    color, depth, sil = img["color"], img["depth"], img["sil"]
    H, W = depth.shape
    dev = depth.device
    if out is None:
        out = (torch.empty_like(color), torch.empty_like(depth), torch.empty_like(sil))
    if loss3 is None:
        loss3 = torch.zeros(3, device=dev)
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_TRACKING_LOSS, 0), dtype=torch.uint8, device=dev)
    _check(lib().csplat_tracking_loss(_ptr(color), _ptr(depth), _ptr(sil), _ptr(obs_color),
                                      _ptr(obs_depth), W, H, lambda_depth, sil_gate,
                                      _ptr(out[0]), _ptr(out[1]), _ptr(out[2]), _ptr(loss3),
                                      _ptr(ws), ws.numel(), _stream(stream)),
           "csplat_tracking_loss")
    return out, loss3


def tile_mask_words(cam: dict) -> int:
    tx, ty = tiles(cam)
    return (tx * ty + 31) // 32


def ba_patches(obs_depth, cam: dict, patches, tile_active=None, n_valid=None, stream=None):
    """NEXT-4: one keyframe's active-tile mask (cleared, then set) and its
    valid-depth rays ADDED to n_valid (device int64[1])."""
    dev = obs_depth.device
    if tile_active is None:
        tile_active = torch.empty(tile_mask_words(cam), dtype=torch.int32, device=dev)
    if n_valid is None:
        n_valid = torch.zeros(1, dtype=torch.int64, device=dev)
    _check(lib().csplat_ba_patches(_ptr(obs_depth), C.byref(camera(cam)), _ptr(patches),
                                   int(patches.numel()), _ptr(tile_active), _ptr(n_valid),
                                   _stream(stream)), "csplat_ba_patches")
    return tile_active, n_valid


def ba_patch_loss(img: dict, obs_color, obs_depth, cam: dict, patches, n_rays: int, n_valid,
                  lambda_depth=1.0, lambda_ssim=0.2, out=None, loss3=None, stream=None):
    """NEXT-4: upstream grads (d_color, d_depth, d_sil) of one keyframe's patches and
    its shares of (L_c, L_d, SSIM) ADDED to loss3 (device float32[3])."""
    color, depth = img["color"], img["depth"]
    dev = depth.device
    if out is None:
        out = (torch.empty_like(color), torch.empty_like(depth), torch.empty_like(depth))
    if loss3 is None:
        loss3 = torch.zeros(3, device=dev)
    _check(lib().csplat_ba_patch_loss(_ptr(color), _ptr(depth), _ptr(obs_color),
                                      _ptr(obs_depth), C.byref(camera(cam)), _ptr(patches),
                                      int(patches.numel()), int(n_rays), _ptr(n_valid),
                                      lambda_depth, lambda_ssim, _ptr(out[0]), _ptr(out[1]),
                                      _ptr(out[2]), _ptr(loss3), _stream(stream)),
           "csplat_ba_patch_loss")
    return out, loss3


def rvq_assign(x, codes, idx_bytes=None, n_dev=None, idx=None, recon=None, want_recon=True,
               stream=None):
    """a2: x [d, n] float32, codes [L, P, d] -> idx [L, n] (uint8/int16), recon [d, n]."""
    d, n = x.shape
    L, P, d2 = codes.shape
    assert d2 == d
    if idx_bytes is None:
        idx_bytes = 1 if P <= 256 else 2
    dev = x.device
    if idx is None:
        idx = torch.empty((L, max(n, 1)), dtype=torch.uint8 if idx_bytes == 1 else torch.int16,
                          device=dev)
    if recon is None and want_recon:
        recon = torch.empty((d, max(n, 1)), device=dev)
    _check(lib().csplat_rvq_assign(_ptr(x), n, _ptr(n_dev), d, _ptr(codes), L, P, _ptr(idx),
                                   idx_bytes, _ptr(recon), _stream(stream)), "csplat_rvq_assign")
    return idx, recon


def rvq_code_grad(d_shat, idx, P: int, n_dev=None, d_codes=None, accumulate=False, stream=None):
    """NEXT-2 STE (reading R31): d_shat [d, n] = dL/dS_hat -> dL/dcodes [L, P, d]."""
    d, n = d_shat.shape
    L = idx.shape[0]
    if d_codes is None:
        d_codes = torch.empty((L, P, d), device=d_shat.device)
    _check(lib().csplat_rvq_code_grad(_ptr(d_shat), n, _ptr(n_dev), d, _ptr(idx),
                                      idx.element_size(), L, P, _ptr(d_codes),
                                      ACCUMULATE if accumulate else 0, _stream(stream)),
           "csplat_rvq_code_grad")
    return d_codes


def rvq_init_stage(x, codes, stage: int, idx, sample, stream=None):
    """NEXT-2 Fig 4 (reading R32): codes[stage] := the stage residuals of x[:, sample]."""
    d, n = x.shape
    L, P = codes.shape[:2]
    ib = idx.element_size() if idx is not None else 1
    _check(lib().csplat_rvq_init_stage(_ptr(x), n, d, _ptr(codes), L, P, stage, _ptr(idx), ib,
                                       _ptr(sample), _stream(stream)), "csplat_rvq_init_stage")
    return codes


def rvq_init(x, L: int, P: int, rng, stream=None):
    """Fig 4: initialise an L-stage, P-code residual codebook on x [d, n]:
    per stage, P vectors drawn without replacement (host rng: the caller's random
    draw) seed the codes with their stage residuals, then the closest-code
    assignment (Eq 10) gives the next stage's residuals.  Returns (codes, idx)."""
    d, n = x.shape
    dev = x.device
    codes = torch.zeros((L, P, d), device=dev)
    idx = torch.zeros((L, n), dtype=torch.uint8 if P <= 256 else torch.int16, device=dev)
    for l in range(L):
        sample = torch.tensor(rng.choice(n, P, replace=False), dtype=torch.int64, device=dev)
        rvq_init_stage(x, codes, l, idx, sample, stream=stream)
        rvq_assign(x, codes[:l + 1], idx=idx[:l + 1], want_recon=False, stream=stream)
    return codes, idx


def mask_loss(g: GaussianMap, count, d_mask, lam=1.0, loss=None, ws=None, stream=None):
    """NEXT-3 (Eq 8 over the in-frustum Gaussians, count > 0): d_mask += lam Sig'(m)/N_a.
    Returns the device loss [1]."""
    dev = g.opacity.device
    if loss is None:
        loss = torch.zeros(1, device=dev)
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_MASK_LOSS, 0), dtype=torch.uint8, device=dev)
    gs = g.struct()
    _check(lib().csplat_mask_loss(C.byref(gs), _ptr(count), lam, _ptr(d_mask), _ptr(loss),
                                  _ptr(ws), ws.numel(), _stream(stream)), "csplat_mask_loss")
    return loss


def keyframe_overlap(depth, cam: dict, cur_view, views, counts=None, ws=None, stream=None):
    """NEXT-3: per keyframe, the number of valid current-depth points inside
    its frustum (device int64 [K]).  views: a list of 4x4/3x4 views, or the
    ctypes array view_array() returns (marshalled once, reused per frame)."""
    K = len(views)
    dev = depth.device
    if counts is None:
        counts = torch.zeros(max(K, 1), dtype=torch.int64, device=dev)
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_KEYFRAME_OVERLAP, K), dtype=torch.uint8, device=dev)
    arr = views if isinstance(views, C.Array) else view_array(views)
    _check(lib().csplat_keyframe_overlap(_ptr(depth), C.byref(camera(cam)), C.byref(view(cur_view)),
                                         arr, K, _ptr(counts), _ptr(ws), ws.numel(),
                                         _stream(stream)), "csplat_keyframe_overlap")
    return counts[:K]


def view_array(views):
    """Marshal a list of views into the csplat_view[K] array keyframe_overlap takes."""
    return (View * max(len(views), 1))(*[view(v) for v in views])


def select_window(overlap_counts, n: int, recency=None):
    """P:138 sliding window: the most relevant keyframe plus the n-2 next by
    overlap (ties -> more recent first); returns keyframe indices (host)."""
    import numpy as np
    c = np.asarray(overlap_counts.cpu() if hasattr(overlap_counts, "cpu") else overlap_counts)
    rec = np.arange(len(c)) if recency is None else np.asarray(recency)
    order = sorted(range(len(c)), key=lambda k: (-int(c[k]), -int(rec[k])))
    return [k for k in order if c[k] > 0][:max(0, n - 1)]


def rvq_update(x, codes, idx, n_dev=None, codes_out=None, want_counts=True, ws=None,
               stream=None):
    """NEXT-2 (Eq 11): k-means M-step of the codebooks for the assignment idx.
    Returns (codes_out [L,P,d], counts [L,P] int32 or None, loss [L+1])."""
    d, n = x.shape
    L, P, _ = codes.shape
    dev = x.device
    if codes_out is None:
        codes_out = torch.empty_like(codes)
    counts = torch.empty((L, P), dtype=torch.int32, device=dev) if want_counts else None
    loss = torch.zeros(L + 1, device=dev)
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_RVQ_UPDATE, L * P, d), dtype=torch.uint8, device=dev)
    _check(lib().csplat_rvq_update(_ptr(x), n, _ptr(n_dev), d, _ptr(codes), L, P, _ptr(idx),
                                   idx.element_size(), _ptr(codes_out), _ptr(counts), _ptr(loss),
                                   _ptr(ws), ws.numel(), _stream(stream)), "csplat_rvq_update")
    return codes_out, counts, loss


def mask_prune(g: GaussianMap, cb: CodebookT | None = None, mask_eps=0.01,
               reset_mask_logit=float("nan"), out: GaussianMap | None = None, out_idx=None,
               keep_map=None, n_kept=None, ws=None, stream=None):
    """a9.  Returns (out GaussianMap with capacity n and n_dev = survivor count, out_idx,
    keep_map, n_kept_dev)."""
    n = g.n
    dev = g.opacity.device
    if out is None:
        out = GaussianMap(**{k: torch.empty_like(getattr(g, k)) for k in
                             ("mean", "opacity", "rgb", "log_scale", "quat", "mask")})
    if cb is not None and out_idx is None:
        out_idx = (torch.empty_like(cb.scale_idx), torch.empty_like(cb.rot_idx))
    if n_kept is None:
        n_kept = torch.zeros(1, dtype=torch.int64, device=dev)
    if ws is None:
        ws = torch.empty(workspace_bytes(OP_MASK_PRUNE, n), dtype=torch.uint8, device=dev)
    o = GaussiansOut(out.n, _ptr(out.mean), _ptr(out.opacity), _ptr(out.rgb),
                     _ptr(out.log_scale), _ptr(out.quat), _ptr(out.mask))
    gs, cbs = g.struct(), cb.struct() if cb is not None else None
    _check(lib().csplat_mask_prune(C.byref(gs), _byref(cbs), mask_eps, reset_mask_logit,
                                   C.byref(o), _ptr(out_idx[0]) if out_idx else None,
                                   _ptr(out_idx[1]) if out_idx else None, _ptr(keep_map),
                                   _ptr(n_kept), _ptr(ws), ws.numel(), _stream(stream)),
           "csplat_mask_prune")
    out.n_dev = n_kept
    return out, out_idx, keep_map, n_kept
