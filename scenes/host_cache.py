"""NumPy producer of the solver's frame planes for CPU-side synthetic scenes
(test and bench data only, not the product path): the reference's
build_cache (frames.py:75-151) - block median depth, block mean luminance,
unprojection, central-difference normals and gradient.  Scenes must be
bit-identical to the reference's to share its goldens; the product path is
the device implementation (`paper_1604_01093_b200.cache.build_cache_device`,
pinned to the same planes by sha256 digests)."""

from __future__ import annotations

import warnings

import numpy as np

from paper_1604_01093_b200.cache import CachedFrame, RgbdFrame
from paper_1604_01093_b200.se3 import Intrinsics


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


