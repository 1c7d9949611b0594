"""Frame caches and correspondence sets: the solver's input records.

`CachedFrame` has the attribute layout of the reference's
`scanfuse.frames.CachedFrame` (frames.py:38-50) and `CorrespondenceSet` that
of `scanfuse.filters.CorrespondenceSet` (filters.py:50-66); the drop-in
solver reads only `valid_depth`, `valid_normal`, `points_low`, `normals_low`,
`grad_low`, `intrinsics_low` and `frame_i/frame_j/points_i/points_j`.

`build_cache_device` is the producer of those planes on the GPU (the
reference's frames.py:75-151, bit-exact); the drop-in `frames.build_cache`
wraps it.  The NumPy restatement used to render CPU-side synthetic scenes
lives outside the product package (`scenes/host_cache.py`).
"""

from __future__ import annotations

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
