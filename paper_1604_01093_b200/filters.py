"""Drop-in `dense_verify` of the reference's correspondence cascade on B200.

Mirrors `scanfuse.filters` (reference filters.py:35-47, 200-277):
`FilterConfig`, `DenseVerifyResult` and `dense_verify(cache_i, cache_j,
transform_ij, config, error_max=None)` keep their names, fields, argument
meaning and pass/fail rule; the two `_verify_one_direction` passes
(filters.py:216-250) run on the GPU, one CTA per direction
(`sfb_dense_verify`, csrc/sfb_verify.cu).  `dense_verify_many` checks a whole
list of frame pairs in one launch - the intra-chunk acceptance check of every
candidate pair (section 3.2: one CTA per frame pair).

Counts are bit-exact with the reference and so is the mean error (NumPy's
pairwise summation is reproduced); `passed` is therefore identical.  There is
no CPU fallback: the CUDA library is required.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi
from ._rounding import probe
from .runtime import runtime

__all__ = ["FilterConfig", "DenseVerifyResult", "dense_verify", "dense_verify_many"]


@dataclass
class FilterConfig:
    """Thresholds of the correspondence cascade (reference filters.py:35-47)."""

    kabsch_residual_max: float = 0.02
    condition_limit: float = 100.0
    min_surface_area: float = 0.032  # m^2
    verify_depth_max: float = 0.15  # point distance gate
    verify_normal_min: float = 0.9  # cosine of normal deviation
    verify_color_max: float = 0.1  # intensity difference gate
    verify_error_max: float = 0.075  # mean reprojection error gate
    verify_min_valid_fraction: float = 0.02  # of w'*h' pixels
    min_correspondences: int = 5
    obb_method: str = "calipers"  # or "pca"


@dataclass
class DenseVerifyResult:
    """reference filters.py:200-213"""

    passed: bool
    mean_error_ij: float
    mean_error_ji: float
    valid_count_ij: int
    valid_count_ji: int

    @property
    def mean_error(self):
        return max(self.mean_error_ij, self.mean_error_ji)

    @property
    def valid_count(self):
        return min(self.valid_count_ij, self.valid_count_ji)


def _f_ordered(rotation) -> bool:
    rot = np.asarray(rotation)
    return bool(rot.flags.f_contiguous and not rot.flags.c_contiguous)


def dense_verify_many(pairs, config: FilterConfig, error_max: float | None = None,
                      device: int | None = None) -> list[DenseVerifyResult]:
    """Dense two-sided check of many relative transforms in one launch.

    `pairs`: iterable of (cache_i, cache_j, transform_ij).  Returns one
    `DenseVerifyResult` per pair, each equal to
    `dense_verify(cache_i, cache_j, transform_ij, config, error_max)`.  The
    j -> i direction uses transform_ij.inverse() evaluated on the device with
    NumPy's rounding (geometry.py:135-137).
    """
    pairs = list(pairs)
    if not pairs:
        return []
    if error_max is None:
        error_max = config.verify_error_max
    rt = runtime(device)
    caches = [c for ci, cj, _ in pairs for c in (ci, cj)]
    slots = np.asarray(rt.intensity_slots_for(caches), dtype=np.int32).reshape(-1, 2)
    n = len(pairs)
    R = np.empty((n, 3, 3), dtype=np.float64)
    t = np.empty((n, 3), dtype=np.float64)
    fo = np.empty(n, dtype=np.uint8)
    for k, (_, _, T) in enumerate(pairs):
        R[k] = T.rotation
        t[k] = T.translation
        fo[k] = 2 if _f_ordered(T.rotation) else 0
    # item 2k: i -> j with transform_ij; item 2k+1: j -> i with its inverse()
    src = np.ascontiguousarray(slots.reshape(-1))
    dst = np.ascontiguousarray(slots[:, ::-1].reshape(-1))
    R9 = np.repeat(R.reshape(n, 9), 2, axis=0)
    t3 = np.repeat(t, 2, axis=0)
    flags = np.repeat(fo, 2)
    flags[1::2] |= 1
    pr = probe()
    cfg = _abi.VerifyConfig(float(config.verify_depth_max), float(config.verify_normal_min),
                            float(config.verify_color_max), pr["apply_n"], pr["apply_1"],
                            pr["apply_nf"], pr["apply_1f"])
    err = np.zeros(2 * n, dtype=np.float64)
    cnt = np.zeros(2 * n, dtype=np.int64)
    with rt.using(src):  # no concurrent clear_frames() may release them mid-call
        _abi.check(rt.lib.sfb_dense_verify(rt.handle, 2 * n, _abi.ptr(src), _abi.ptr(dst),
                                           _abi.ptr(R9), _abi.ptr(t3), _abi.ptr(flags),
                                           _abi.C.byref(cfg), _abi.ptr(err), _abi.ptr(cnt)),
                   rt.handle)
    out = []
    for k, (ci, _, _) in enumerate(pairs):
        err_ij, err_ji = float(err[2 * k]), float(err[2 * k + 1])
        count_ij, count_ji = int(cnt[2 * k]), int(cnt[2 * k + 1])
        kl = ci.intrinsics_low
        min_count = config.verify_min_valid_fraction * kl.width * kl.height  # filters.py:270
        passed = (count_ij >= min_count and count_ji >= min_count and err_ij <= error_max
                  and err_ji <= error_max)
        out.append(DenseVerifyResult(bool(passed), err_ij, err_ji, count_ij, count_ji))
    return out


def dense_verify(cache_i, cache_j, transform_ij, config: FilterConfig,
                 error_max: float | None = None) -> DenseVerifyResult:
    """Two-sided dense consistency check of a relative transform
    (reference filters.py:253-277): each valid pixel of one frame is
    reprojected into the other and counts when point distance, normal
    deviation and intensity difference all pass their gates; the pair passes
    when both directions keep enough pixels and their mean error stays at or
    below `error_max` (default `config.verify_error_max`)."""
    return dense_verify_many([(cache_i, cache_j, transform_ij)], config, error_max)[0]
