"""Drop-in for the solver-facing part of `scanfuse.frames` (reference frames.py).

* `CachedFrame`, `RgbdFrame`: the reference's records (frames.py:27-50).
* `build_cache(frame, intrinsics, low_width, low_height)` (frames.py:75-123):
  the device kernels of `cache.build_cache_device` for one frame; the planes
  stay resident in the device frame store.
* `frustum_overlap` (frames.py:154-180): the pair filter's exact per-point
  kernel (`sfb_frustum_overlap`), bit-exact with NumPy's rounding.
* `view_angle_deg` (frames.py:183-188): a three-term dot of two rotation
  columns, evaluated on the host exactly as the reference does (it is the
  scalar the device pair filter's angle gate reproduces, see
  `device_problem.view_cos_threshold`).
"""

from __future__ import annotations

import numpy as np

from .cache import CachedFrame, RgbdFrame, build_cache_device

__all__ = ["CachedFrame", "RgbdFrame", "build_cache", "frustum_overlap", "view_angle_deg"]


def build_cache(frame: RgbdFrame, intrinsics, low_width: int = 80, low_height: int = 60,
                device: int | None = None) -> CachedFrame:
    """Downsampled working copy of one frame, built on the GPU (frames.py:75-123)."""
    return build_cache_device([frame], intrinsics, low_width, low_height, device)[0]


def frustum_overlap(cache_a, pose_a, cache_b, pose_b) -> float:
    """Fraction of a's valid cached points that land inside b's view (frames.py:154-180)."""
    from .device_problem import DeviceProblem
    if not np.any(np.asarray(cache_a.valid_depth)):
        return 0.0
    dp = DeviceProblem(2, [cache_a, cache_b])
    try:
        dp.set_poses([pose_a, pose_b])
        return float(dp.frustum_overlap([(0, 1)])[0])
    finally:
        dp.close()


def view_angle_deg(pose_a, pose_b) -> float:
    """Angle in degrees between the two cameras' viewing directions (frames.py:183-188)."""
    za = np.asarray(pose_a.rotation)[:, 2]
    zb = np.asarray(pose_b.rotation)[:, 2]
    cosang = np.clip(np.dot(za, zb), -1.0, 1.0)
    return float(np.degrees(np.arccos(cosang)))
