"""Frame caches and correspondence sets: the solver's input records.

`CachedFrame` has the attribute layout of the reference's
`scanfuse.frames.CachedFrame` (frames.py:38-50) and `CorrespondenceSet` that
of `scanfuse.filters.CorrespondenceSet` (filters.py:50-66); the drop-in
solver reads only `valid_depth`, `valid_normal`, `points_low`, `normals_low`,
`grad_low`, `intrinsics_low` and `frame_i/frame_j/points_i/points_j`.

`build_cache` is the host-side producer of those planes (the reference's
frames.py:75-151: block median depth, block mean luminance, unprojection,
central-difference normals and gradient); it is upstream of the solver hot
path and is used here to build synthetic scenes.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np

from .se3 import Intrinsics, RigidTransform

LUMA = np.array([0.299, 0.587, 0.114])


@dataclass
class RgbdFrame:
    index: int
    color: np.ndarray   # (H, W, 3) uint8
    depth: np.ndarray   # (H, W) float32 meters, 0 = invalid
    timestamp: float = 0.0

    def luminance(self) -> np.ndarray:
        return (self.color.astype(np.float32) @ LUMA.astype(np.float32)) / 255.0


@dataclass
class CachedFrame:
    index: int
    intensity_low: np.ndarray
    grad_low: np.ndarray
    depth_low: np.ndarray
    points_low: np.ndarray
    normals_low: np.ndarray
    intrinsics_low: Intrinsics
    valid_depth: np.ndarray = field(repr=False, default=None)
    valid_normal: np.ndarray = field(repr=False, default=None)


@dataclass
class CorrespondenceSet:
    frame_i: int
    frame_j: int
    points_i: np.ndarray
    points_j: np.ndarray
    indices: np.ndarray = None
    transform: RigidTransform = None
    valid: bool = False

    def __len__(self):
        return self.points_i.shape[0]


def _blocks(a: np.ndarray, bh: int, bw: int) -> np.ndarray:
    h, w = a.shape
    return a.reshape(h // bh, bh, w // bw, bw).transpose(0, 2, 1, 3).reshape(h // bh, w // bw, -1)


def _median_valid(depth: np.ndarray, bh: int, bw: int) -> np.ndarray:
    blk = _blocks(depth, bh, bw)
    bad = blk <= 0.0
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        med = np.nanmedian(np.where(bad, np.nan, blk), axis=2)
    out = np.zeros(blk.shape[:2], dtype=np.float32)
    keep = ~np.all(bad, axis=2)
    out[keep] = med[keep].astype(np.float32)
    return out


def normals_from_points(points: np.ndarray, valid: np.ndarray):
    """Central-difference normals facing the camera (frames.py:126-151)."""
    h, w = valid.shape
    ok = np.zeros((h, w), dtype=bool)
    ok[1:-1, 1:-1] = (valid[1:-1, 1:-1] & valid[1:-1, 2:] & valid[1:-1, :-2]
                      & valid[2:, 1:-1] & valid[:-2, 1:-1])
    gx = np.zeros((h, w, 3), dtype=np.float32)
    gy = np.zeros((h, w, 3), dtype=np.float32)
    gx[1:-1, 1:-1] = points[1:-1, 2:] - points[1:-1, :-2]
    gy[1:-1, 1:-1] = points[2:, 1:-1] - points[:-2, 1:-1]
    n = np.cross(gy.reshape(-1, 3), gx.reshape(-1, 3)).reshape(h, w, 3)
    ln = np.linalg.norm(n, axis=-1)
    ok &= ln > 1e-12
    n[ok] /= ln[ok][..., None]
    towards = np.sum(n * points, axis=-1) > 0.0
    n[towards & ok] *= -1.0
    n[~ok] = 0.0
    out = np.zeros((h, w, 3), dtype=np.float32)
    out[:] = n
    return out, ok


def build_cache(frame: RgbdFrame, intrinsics: Intrinsics, low_width: int = 80,
                low_height: int = 60) -> CachedFrame:
    h, w = frame.depth.shape
    if h % low_height or w % low_width:
        raise ValueError(f"frame {w}x{h} does not divide into {low_width}x{low_height} blocks")
    bh, bw = h // low_height, w // low_width
    lum = frame.luminance()
    intensity = lum.reshape(h // bh, bh, w // bw, bw).mean(axis=(1, 3)).astype(np.float32)
    depth = _median_valid(frame.depth.astype(np.float32), bh, bw)
    k = intrinsics.scaled(low_width, low_height)
    xs, ys = np.meshgrid(np.arange(low_width), np.arange(low_height))
    valid = depth > 0.0
    pts = k.unproject(np.stack([xs, ys], axis=-1).astype(np.float64),
                      depth.astype(np.float64)).astype(np.float32)
    pts[~valid] = 0.0
    nrm, valid_n = normals_from_points(pts, valid)
    grad = np.zeros((low_height, low_width, 2), dtype=np.float32)
    grad[:, 1:-1, 0] = 0.5 * (intensity[:, 2:] - intensity[:, :-2])
    grad[1:-1, :, 1] = 0.5 * (intensity[2:, :] - intensity[:-2, :])
    return CachedFrame(frame.index, intensity, grad, depth, pts, nrm, k, valid, valid_n)


def build_cache_device(frames, intrinsics: Intrinsics, low_width: int = 80, low_height: int = 60,
                       device: int | None = None) -> list:
    """`build_cache` for a batch of frames on the GPU (one launch pair).

    Returns one `CachedFrame` per `RgbdFrame`, every plane bit-identical to
    the reference's build_cache (frames.py:75-151).  The planes stay resident
    in the device frame store, so solving or verifying with these caches
    uploads nothing.  All frames must share one resolution; blocks of at
    most 64 samples (e.g. 640x480 -> 80x60).
    """
    import ctypes as C

    from . import _abi
    from ._rounding import probe_luma
    from .runtime import runtime

    frames = list(frames)
    if not frames:
        return []
    h, w = np.asarray(frames[0].depth).shape
    if h % low_height or w % low_width:
        raise ValueError(f"frame {w}x{h} does not divide into {low_width}x{low_height} blocks")
    cols, deps = [], []
    for f in frames:
        col = np.ascontiguousarray(f.color, dtype=np.uint8)
        dep = np.ascontiguousarray(f.depth, dtype=np.float32)
        if col.shape != (h, w, 3) or dep.shape != (h, w):
            raise ValueError("all frames of a batch must share one resolution")
        cols.append(col)
        deps.append(dep)
    k = intrinsics.scaled(low_width, low_height)
    k4 = np.array([k.fx, k.fy, k.cx, k.cy], dtype=np.float64)
    n = len(frames)
    hw = low_width * low_height
    out = np.empty(n * 42 * hw, dtype=np.uint8)
    slots = np.zeros(n, dtype=np.int32)
    rt = runtime(device)
    cp = (C.c_void_p * n)(*[a.ctypes.data for a in cols])
    dp = (C.c_void_p * n)(*[a.ctypes.data for a in deps])
    _abi.check(rt.lib.sfb_build_cache(rt.handle, n, w, h, low_width, low_height, cp, dp,
                                      _abi.ptr(k4), probe_luma(), _abi.ptr(out), _abi.ptr(slots)),
               rt.handle)
    res = []
    shp = (low_height, low_width)
    for i, f in enumerate(frames):
        b = out[i * 42 * hw:(i + 1) * 42 * hw]
        f32 = b[:40 * hw].view(np.float32)
        intensity = f32[:hw].reshape(shp)
        depth = f32[hw:2 * hw].reshape(shp)
        pts = f32[2 * hw:5 * hw].reshape(shp + (3,))
        nrm = f32[5 * hw:8 * hw].reshape(shp + (3,))
        grad = f32[8 * hw:10 * hw].reshape(shp + (2,))
        vd = b[40 * hw:41 * hw].view(np.bool_).reshape(shp)
        vn = b[41 * hw:42 * hw].view(np.bool_).reshape(shp)
        res.append(CachedFrame(f.index, intensity, grad, depth, pts, nrm, k, vd, vn))
    rt.adopt(res, slots)
    return res
