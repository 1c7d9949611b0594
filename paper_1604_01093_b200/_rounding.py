"""Probe how this host's NumPy/BLAS rounds the 3-term products the reference uses.

The frame-pair filter must select exactly the pairs the reference selects
(build_dense_edges, solver.py:130-148), and its decisions go through
`RigidTransform.inverse/compose/apply` (geometry.py:127-151) and `np.dot`
(frames.py:187), which NumPy hands to OpenBLAS.  OpenBLAS evaluates every
3-term dot as an FMA chain whose order depends on the kernel it picked for
this CPU (DYNAMIC_ARCH) and on the memory layout.  We measure the order once
per process against exact rational arithmetic and pass it to the kernels.

Order code o -> first product a_i*b_i, then fma(a_j,b_j,.), then fma(a_k,b_k,.):
0:(0,1,2) 1:(0,2,1) 2:(1,0,2) 3:(1,2,0) 4:(2,0,1) 5:(2,1,0)
"""

from __future__ import annotations

import functools
import warnings
from fractions import Fraction

import numpy as np

PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
DEFAULT = dict(matvec_c=2, matvec_f=0, gemm33=0, apply_n=0, apply_1=2, dot3=0,
               apply_nf=0, apply_1f=2)


def _fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def chain(a, b, code: int) -> float:
    i, j, k = PERMS[code]
    return _fma(a[k], b[k], _fma(a[j], b[j], float(Fraction(a[i]) * Fraction(b[i]))))


def _survivors(trials, fn, rng) -> set:
    alive = set(range(6))
    for _ in range(trials):
        a = rng.normal(size=3) * rng.uniform(0.1, 10.0)
        b = rng.normal(size=3) * rng.uniform(0.1, 10.0)
        got = fn(a, b, rng)
        alive &= {o for o in range(6) if chain(a, b, o) == got}
        if not alive:
            break
    return alive


def _mv_c(a, b, rng):
    M = rng.normal(size=(3, 3))
    M[1] = a
    return float((M @ b)[1])


def _mv_f(a, b, rng):
    M = np.asfortranarray(rng.normal(size=(3, 3)))
    M[1] = a
    return float((M @ b)[1])


def _gemm(a, b, rng):
    A = rng.normal(size=(3, 3))
    B = rng.normal(size=(3, 3))
    A[2] = a
    B[:, 0] = b
    return float((A @ B)[2, 0])


def _apply_n(a, b, rng):
    P = rng.normal(size=(64, 3))
    R = rng.normal(size=(3, 3))
    P[17] = a
    R[2] = b
    return float((P @ R.T)[17, 2])


def _apply_1(a, b, rng):
    R = rng.normal(size=(3, 3))
    R[0] = b
    return float((a[None, :] @ R.T)[0, 0])


def _apply_nf(a, b, rng):  # Fortran-ordered rotation (dense_verify's caller transform)
    P = rng.normal(size=(64, 3))
    R = np.asfortranarray(rng.normal(size=(3, 3)))
    P[17] = a
    R[2] = b
    return float((P @ R.T)[17, 2])


def _apply_1f(a, b, rng):
    R = np.asfortranarray(rng.normal(size=(3, 3)))
    R[0] = b
    return float((a[None, :] @ R.T)[0, 0])


def _dot(a, b, rng):
    return float(np.dot(a, b))


LUMA = (0.299, 0.587, 0.114)


@functools.lru_cache(maxsize=1)
def probe_luma() -> int:
    """FMA chain order of RgbdFrame.luminance (frames.py:33-35):
    (H,W,3) float32 @ (3,) float32, on this host's NumPy/BLAS.  Returns the
    order code with the fewest mismatches over random 8-bit colours (the
    float64 emulation of a float32 FMA double-rounds in rare ties)."""
    rng = np.random.default_rng(33)
    col = rng.integers(0, 256, size=(32, 96, 3), dtype=np.uint8).astype(np.float32)
    w = np.array(LUMA).astype(np.float32)
    got = col @ w
    c = col.reshape(-1, 3).astype(np.float64)
    wd = w.astype(np.float64)
    best, best_bad = 0, None
    for code, (i, j, k) in enumerate(PERMS):
        r = (c[:, i] * wd[i]).astype(np.float32).astype(np.float64)
        r = (c[:, j] * wd[j] + r).astype(np.float32).astype(np.float64)
        r = (c[:, k] * wd[k] + r).astype(np.float32)
        bad = int(np.count_nonzero(r != got.reshape(-1)))
        if best_bad is None or bad < best_bad:
            best, best_bad = code, bad
    return best


@functools.lru_cache(maxsize=1)
def probe(trials: int = 300) -> dict:
    rng = np.random.default_rng(20160404)
    out = {}
    for name, fn in (("matvec_c", _mv_c), ("matvec_f", _mv_f), ("gemm33", _gemm),
                     ("apply_n", _apply_n), ("apply_1", _apply_1), ("dot3", _dot),
                     ("apply_nf", _apply_nf), ("apply_1f", _apply_1f)):
        alive = _survivors(trials, fn, rng)
        if alive:
            out[name] = DEFAULT[name] if DEFAULT[name] in alive else min(alive)
        else:
            warnings.warn(f"NumPy {name} rounding matches no FMA chain; using default order "
                          "(pair-filter decisions at exact ties may differ)")
            out[name] = DEFAULT[name]
    return out
