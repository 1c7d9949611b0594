"""Drop-in, B200-native replacement for `scanfuse.solver` (reference solver.py).

Same public names, signatures, data layouts and error behaviour as the
reference module; every numeric step runs in libsfb.so on the GPU:

* `AlignmentProblem.solve` (solver.py:681-750) keeps the reference's
  Gauss-Newton control flow on the host (dense ramp, accept / two-strike
  abort / best-pose restore, relative-decrease convergence) and only moves
  scalars across PCIe per iteration; linearisation, the block system, the
  scalar-Jacobi PCG, the Lie update and the frozen-association energy are
  device kernels.
* `build_dense_edges` (:130-148) is the bit-exact device pair filter.
* `pcg_solve` (:463-508) runs the exact recurrence on the device; it stays
  duck-typed: a foreign system exposing `.rhs/.diagonal/.apply` is
  materialised through its own `apply` and solved by the same device PCG.
* The per-edge evaluators (:114-349) return host arrays computed on device.

There is no CPU fallback: without libsfb.so or a CUDA device every entry
point raises.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import operator
import threading

import numpy as np

from . import _abi
from .device_problem import DeviceProblem, _host_module
from .runtime import runtime
from .se3 import RigidTransform


class PcgDivergenceError(RuntimeError):
    """Non-finite values appeared inside the linear solve (solver.py:30-31)."""


@dataclass
class EnergyWeights:
    sparse: float = 1.0
    photo: float = 0.1
    geo: float = 1.0
    dense_ramp: tuple = (0, 5)


def dense_ramp_weight(weights: EnergyWeights, iteration: int) -> float:
    """Linear 0 -> 1 dense-term ramp over outer iterations (solver.py:49-53)."""
    start, end = weights.dense_ramp
    if end <= start:
        return 1.0 if iteration >= end else 0.0
    return float(np.clip((iteration - start) / (end - start), 0.0, 1.0))


@dataclass
class SolverConfig:
    batch_iterations: int = 10
    online_iterations: int = 3
    pcg_max_iterations: int = 50
    pcg_tolerance: float = 1e-6
    pcg_restart_interval: int = 20
    min_relative_decrease: float = 1e-9
    view_angle_max_deg: float = 60.0
    geo_distance_max: float = 0.15
    geo_normal_min: float = 0.9
    dense_pixel_stride: int = 1
    dense_bidirectional: bool = False
    prune_residual_max: float = 0.05
    # PCG preconditioner (not a reference field): "jacobi" is the reference's
    # scalar Jacobi (solver.py:477); "block_jacobi" (opt-in performance mode)
    # inverts each frame's 6x6 diagonal block and does NOT reproduce the
    # reference's iterates.
    preconditioner: str = "jacobi"


_PRECONDITIONERS = {"jacobi": 0, "block_jacobi": 1}


def _precond_kind(config) -> int:
    name = getattr(config, "preconditioner", "jacobi")
    if name not in _PRECONDITIONERS:
        raise ValueError(f"unknown preconditioner {name!r} (expected one of {sorted(_PRECONDITIONERS)})")
    return _PRECONDITIONERS[name]


# ---------------------------------------------------------------------------
# Sparse term


@dataclass
class SparseTerm:
    """Stacked correspondences with variable indices, -1 = anchor (solver.py:76-86)."""

    var_i: np.ndarray
    var_j: np.ndarray
    points_i: np.ndarray
    points_j: np.ndarray
    set_index: np.ndarray
    frames_i: np.ndarray
    frames_j: np.ndarray


def build_sparse_term(corr_sets, frame_to_var) -> SparseTerm:
    """Host packing of CorrespondenceSets into SoA (solver.py:89-111)."""
    if not corr_sets:
        e = np.zeros(0, dtype=int)
        return SparseTerm(e, e, np.zeros((0, 3)), np.zeros((0, 3)), e, e, e)
    sizes = np.array([len(cs) for cs in corr_sets], dtype=int)
    fi = np.array([cs.frame_i for cs in corr_sets])
    fj = np.array([cs.frame_j for cs in corr_sets])
    vi = np.array([frame_to_var[f] for f in fi], dtype=int)
    vj = np.array([frame_to_var[f] for f in fj], dtype=int)
    pts_i = np.vstack([np.asarray(cs.points_i, dtype=np.float64).reshape(-1, 3) for cs in corr_sets])
    pts_j = np.vstack([np.asarray(cs.points_j, dtype=np.float64).reshape(-1, 3) for cs in corr_sets])
    return SparseTerm(np.repeat(vi, sizes), np.repeat(vj, sizes), pts_i, pts_j,
                      np.repeat(np.arange(len(corr_sets)), sizes), np.repeat(fi, sizes),
                      np.repeat(fj, sizes))


_get_fi = operator.attrgetter("frame_i")
_get_fj = operator.attrgetter("frame_j")
_get_pi = operator.attrgetter("points_i")
_get_pj = operator.attrgetter("points_j")
_get_dtype = operator.attrgetter("dtype")


def _set_layout_native(corr_sets, frame_index, rt):
    """_set_layout in C (_sfbhost.stack_sets_into) into the runtime's reusable
    page-locked staging buffers; None when the sets need the NumPy path.  The
    returned arrays alias staging memory: consume them before the next call."""
    try:
        from . import _sfbhost
    except ImportError:
        return None
    n = len(corr_sets)
    fr = rt.staging("sets_frames", 8 * n).view(np.int32)
    of = rt.staging("sets_offsets", 8 * (n + 1)).view(np.int64)
    rows = 1 << 14
    for _ in range(2):
        pi = rt.staging("sets_pi", 24 * rows).view(np.float64)
        pj = rt.staging("sets_pj", 24 * rows).view(np.float64)
        r = _sfbhost.stack_sets_into(corr_sets, frame_index, fr, of, pi, pj)
        if r is None:
            return None
        if r >= 0:
            return (fr[:2 * n].reshape(n, 2), of[:n + 1], pi[:3 * r].reshape(r, 3),
                    pj[:3 * r].reshape(r, 3))
        rows = -r - 1  # grow to the reported size and redo
    return None


def _set_layout(corr_sets, frame_index, rt=None):
    """(n_sets,2) problem-frame indices, offsets and stacked points for the ABI
    (build_sparse_term's stacking, solver.py:89-111).  With a runtime `rt`, the
    C stacker writes into its reusable pinned staging (consume immediately)."""
    n = len(corr_sets)
    if n == 0:
        return (np.zeros((0, 2), dtype=np.int32), np.zeros(1, dtype=np.int64), np.zeros((0, 3)),
                np.zeros((0, 3)))
    if rt is not None:
        lay = _set_layout_native(corr_sets, frame_index, rt)
        if lay is not None:
            return lay
    fi = np.fromiter(map(_get_fi, corr_sets), dtype=np.int64, count=n)
    fj = np.fromiter(map(_get_fj, corr_sets), dtype=np.int64, count=n)
    keys = np.fromiter(frame_index.keys(), dtype=np.int64, count=len(frame_index))
    vals = np.fromiter(frame_index.values(), dtype=np.int64, count=len(frame_index))
    if keys.size and keys.min() >= 0 and keys.max() < 16 * keys.size + 1024:
        lut = np.full(int(keys.max()) + 1, -1, dtype=np.int64)
        lut[keys] = vals
        ok_ids = (fi >= 0) & (fi < lut.size) & (fj >= 0) & (fj < lut.size)
        if not ok_ids.all():
            raise KeyError("correspondence set references a frame outside the problem")
        fi, fj = lut[fi], lut[fj]
        if (fi < 0).any() or (fj < 0).any():
            raise KeyError("correspondence set references a frame outside the problem")
    else:
        fi = np.fromiter((frame_index[int(f)] for f in fi), dtype=np.int64, count=n)
        fj = np.fromiter((frame_index[int(f)] for f in fj), dtype=np.int64, count=n)
    frames = np.stack([fi, fj], axis=1).astype(np.int32)
    pi = list(map(_get_pi, corr_sets))
    pj = list(map(_get_pj, corr_sets))
    si = np.fromiter(map(len, pi), dtype=np.int64, count=n)
    sj = np.fromiter(map(len, pj), dtype=np.int64, count=n)
    tot = int(si.sum())
    pts_i = pts_j = None
    try:
        # fast path: one C-level join of the raw buffers (about 2x faster than
        # np.concatenate); requires float64 arrays (checked), C-contiguous
        # (bytes.join raises BufferError otherwise) and (k, 3) (byte count)
        if set(map(_get_dtype, pi)) | set(map(_get_dtype, pj)) == {np.dtype(np.float64)}:
            bi, bj = b"".join(pi), b"".join(pj)
            if len(bi) == 24 * tot and len(bj) == 24 * int(sj.sum()):
                pts_i = np.frombuffer(bi, dtype=np.float64).reshape(-1, 3)
                pts_j = np.frombuffer(bj, dtype=np.float64).reshape(-1, 3)
    except (AttributeError, TypeError, BufferError, ValueError):
        pts_i = pts_j = None
    if pts_i is None:
        pi = [np.asarray(cs, dtype=np.float64).reshape(-1, 3) for cs in pi]
        pj = [np.asarray(cs, dtype=np.float64).reshape(-1, 3) for cs in pj]
        si = np.fromiter((a.shape[0] for a in pi), dtype=np.int64, count=n)
        sj = np.fromiter((b.shape[0] for b in pj), dtype=np.int64, count=n)
        pts_i, pts_j = np.concatenate(pi), np.concatenate(pj)
    if not np.array_equal(si, sj):
        raise ValueError("points_i and points_j of a correspondence set differ in shape")
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(si, out=off[1:])
    return frames, off, np.ascontiguousarray(pts_i), np.ascontiguousarray(pts_j)


def _poses_from_arrays(R, t):
    return [RigidTransform(R[k].copy(), t[k].copy()) for k in range(R.shape[0])]


def _sparse_problem(poses: dict, corr_sets):
    ids = list(dict.fromkeys(f for cs in corr_sets for f in (cs.frame_i, cs.frame_j)))
    index = {f: k for k, f in enumerate(ids)}
    frames, off, pi, pj = _set_layout(corr_sets, index)
    dp = DeviceProblem(max(1, len(ids)), None, frames, pi, pj, off)
    if ids:
        dp.set_poses([poses[f] for f in ids])
    return dp


def eval_sparse(poses: dict, corr_sets):
    """Residuals T_i p_i - T_j p_j (n,3) and their summed square (solver.py:114-123)."""
    if not corr_sets:
        return np.zeros((0, 3)), 0.0
    dp = _sparse_problem(poses, corr_sets)
    res = dp.sparse_residuals()
    dp.close()
    return res, float(np.sum(res ** 2))


# ---------------------------------------------------------------------------
# Dense terms


def _pair_problem(poses, frame_i, frame_j, cache_i, cache_j):
    dp = DeviceProblem(2, [cache_i, cache_j])
    dp.set_poses([poses[frame_i], poses[frame_j]])
    return dp


def build_dense_edges(frame_ids, poses, caches, config: SolverConfig):
    """Frame pairs admitted to the dense terms (solver.py:130-148), on device, bit-exact."""
    ids = list(frame_ids)
    if len(ids) < 2:
        return []
    dp = DeviceProblem(len(ids), [caches[f] for f in ids])
    dp.set_poses([poses[f] for f in ids])
    pairs = dp.build_dense_edges(config.view_angle_max_deg)
    dp.close()
    return [(ids[a], ids[b]) for a, b in pairs]


def _directed_edges(edges, bidirectional):
    directed = list(edges)
    if bidirectional:
        directed += [(j, i) for (i, j) in edges]
    return directed


@dataclass
class PhotoAssociation:
    frame_i: int
    frame_j: int
    points: np.ndarray     # (m,3) source camera-space points
    reference: np.ndarray  # (m,2) gradient at the source pixels


@dataclass
class GeoAssociation:
    frame_i: int
    frame_j: int
    points: np.ndarray
    normals: np.ndarray
    targets: np.ndarray


def _cfg_stride(stride, config=None):
    cfg = config if config is not None else SolverConfig()
    return _StrideConfig(cfg, stride)


class _StrideConfig:
    def __init__(self, cfg, stride):
        self.geo_distance_max = cfg.geo_distance_max
        self.geo_normal_min = cfg.geo_normal_min
        self.dense_pixel_stride = int(stride)
        self.dense_bidirectional = False


def associate_photo(poses, frame_i, frame_j, cache_i, cache_j, stride=1):
    """Source pixels whose warp lands inside frame j (solver.py:216-232)."""
    dp = _pair_problem(poses, frame_i, frame_j, cache_i, cache_j)
    sel, _ = dp.associate(0, 1, 0, _cfg_stride(stride))
    dp.close()
    ys, xs = np.nonzero(sel.reshape(np.asarray(cache_i.valid_depth).shape))
    return PhotoAssociation(frame_i, frame_j,
                            np.asarray(cache_i.points_low)[ys, xs].astype(np.float64),
                            np.asarray(cache_i.grad_low)[ys, xs].astype(np.float64))


def associate_geo(poses, frame_i, frame_j, cache_i, cache_j, config: SolverConfig, stride=1):
    """Projective association with distance/normal gates (solver.py:235-260)."""
    dp = _pair_problem(poses, frame_i, frame_j, cache_i, cache_j)
    sel, tgt = dp.associate(0, 1, 1, _cfg_stride(stride, config))
    dp.close()
    shape = np.asarray(cache_i.valid_depth).shape
    ys, xs = np.nonzero(sel.reshape(shape))
    t = tgt.reshape(shape)[ys, xs]
    wj = np.asarray(cache_j.valid_depth).shape[1]
    ty, tx = t // wj, t % wj
    return GeoAssociation(frame_i, frame_j,
                          np.asarray(cache_i.points_low)[ys, xs].astype(np.float64),
                          np.asarray(cache_i.normals_low)[ys, xs].astype(np.float64),
                          np.asarray(cache_j.points_low)[ty, tx].astype(np.float64))


def photo_residuals(poses, assoc: PhotoAssociation, cache_j):
    """ref - I_j(pi(T_j^-1 T_i d)) on a frozen association (solver.py:263-274)."""
    if assoc.points.shape[0] == 0:
        return np.zeros((0, 2))
    dp = _pair_problem(poses, assoc.frame_i, assoc.frame_j, cache_j, cache_j)
    res, _ = dp.point_eval(0, 1, 0, assoc.points, assoc.reference, jacobian=False)
    dp.close()
    return res


def _nocache_pair(poses, frame_i, frame_j):
    dp = DeviceProblem(2, None)
    dp.set_poses([poses[frame_i], poses[frame_j]])
    return dp


def geo_residuals(poses, assoc: GeoAssociation):
    """n . (d - T_i^-1 T_j target) on a frozen association (solver.py:277-283)."""
    if assoc.points.shape[0] == 0:
        return np.zeros(0)
    dp = _nocache_pair(poses, assoc.frame_i, assoc.frame_j)
    res, _ = dp.point_eval(0, 1, 1, assoc.points, assoc.normals, assoc.targets, jacobian=False)
    dp.close()
    return res


def photo_linearize(poses, assoc: PhotoAssociation, cache_j):
    """Residuals and analytic J_i, J_j = -J_i of a photo edge (solver.py:286-310)."""
    m = assoc.points.shape[0]
    if m == 0:
        return np.zeros((0, 2)), np.zeros((0, 2, 6)), np.zeros((0, 2, 6))
    dp = _pair_problem(poses, assoc.frame_i, assoc.frame_j, cache_j, cache_j)
    res, J = dp.point_eval(0, 1, 0, assoc.points, assoc.reference)
    dp.close()
    return res, J, -J


def geo_linearize(poses, assoc: GeoAssociation):
    """Residuals and analytic J_i, J_j = -J_i of a geo edge (solver.py:313-328)."""
    m = assoc.points.shape[0]
    if m == 0:
        return np.zeros(0), np.zeros((0, 6)), np.zeros((0, 6))
    dp = _nocache_pair(poses, assoc.frame_i, assoc.frame_j)
    res, J = dp.point_eval(0, 1, 1, assoc.points, assoc.normals, assoc.targets)
    dp.close()
    return res, J, -J


def eval_photo(poses, edges, caches, stride=1):
    """Photo residuals over directed edges, fresh association (solver.py:331-338)."""
    residuals = [photo_residuals(poses, associate_photo(poses, i, j, caches[i], caches[j], stride),
                                 caches[j]) for (i, j) in edges]
    res = np.vstack(residuals) if residuals else np.zeros((0, 2))
    return res, float(np.sum(res ** 2))


def eval_geo(poses, edges, caches, config: SolverConfig = None, stride=1):
    """Geo residuals over directed edges, fresh association (solver.py:341-349)."""
    config = config or SolverConfig()
    residuals = [geo_residuals(poses, associate_geo(poses, i, j, caches[i], caches[j], config,
                                                    stride)) for (i, j) in edges]
    res = np.concatenate(residuals) if residuals else np.zeros(0)
    return res, float(np.sum(res ** 2))


# ---------------------------------------------------------------------------
# Normal equations


class NormalEquations:
    """Device-resident Gauss-Newton system (solver.py:356-454).

    Holds the 6x6 block system assembled on the GPU by `normal_equations`.
    Host accessors download on demand; `apply` runs the device block matvec.
    The object is a view of its problem's current linearisation: re-linearising
    the problem invalidates it.
    """

    def __init__(self, device_problem: DeviceProblem, n_vars: int, w_sparse: float,
                 var_i: np.ndarray, var_j: np.ndarray):
        self._dp = device_problem
        self._version = device_problem.version
        self.n_vars = n_vars
        self.w_sparse = w_sparse
        self.var_i = var_i
        self.var_j = var_j
        self._cache = {}

    def _live(self) -> DeviceProblem:
        if self._dp.version != self._version or self._dp.handle is None:
            raise RuntimeError("NormalEquations is stale: its problem was re-linearised")
        return self._dp

    def _get(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    @property
    def gradient(self) -> np.ndarray:
        return self._get("g", lambda: self._live().gradient())

    @property
    def rhs(self) -> np.ndarray:
        return -self.gradient

    @property
    def diagonal(self) -> np.ndarray:
        return self._get("d", lambda: self._live().diagonal())

    @property
    def world_i(self):
        return self._get("w", lambda: self._live().sparse_world())[0]

    @property
    def world_j(self):
        return self._get("w", lambda: self._live().sparse_world())[1]

    def apply(self, x):
        """(J^T J) x on the device (solver.py:403-410)."""
        x = np.asarray(x, dtype=np.float64)
        if self.n_vars == 0:
            return np.zeros(0)
        return self._live().matvec(x)

    def materialize_sparse_jacobian(self):
        """Explicit (3n, N) sparse-term Jacobian (solver.py:430-444), small problems only."""
        wi, wj = self.world_i, self.world_j
        n = wi.shape[0]
        J = np.zeros((3 * n, self.n_vars))
        for k in range(n):
            r = slice(3 * k, 3 * k + 3)
            for var, y, sgn in ((self.var_i[k], wi[k], 1.0), (self.var_j[k], wj[k], -1.0)):
                if var >= 0:
                    c = 6 * var
                    J[r, c:c + 3] += -sgn * np.array([[0.0, -y[2], y[1]], [y[2], 0.0, -y[0]],
                                                      [-y[1], y[0], 0.0]])
                    J[r, c + 3:c + 6] += sgn * np.eye(3)
        return J

    def materialize(self):
        """Full matrix from the device blocks (small problems only)."""
        D, B, pv = self._get("b", lambda: self._live().blocks())
        A = np.zeros((self.n_vars, self.n_vars))
        for v in range(D.shape[0]):
            A[6 * v:6 * v + 6, 6 * v:6 * v + 6] = D[v]
        for q, (a, b) in enumerate(pv):
            A[6 * a:6 * a + 6, 6 * b:6 * b + 6] += B[q]
            A[6 * b:6 * b + 6, 6 * a:6 * a + 6] += B[q].T
        return A

    @property
    def dense_jtj(self):
        """Dense-term part of the system (the reference's precomputed matrix)."""
        A = self.materialize()
        if self.world_i.shape[0] and self.w_sparse > 0.0:
            J = self.materialize_sparse_jacobian()
            A = A - self.w_sparse * (J.T @ J)
        return A


@dataclass
class PcgResult:
    iterations: int
    relative_residual: float


def pcg_solve(equations, max_iterations: int = 50, tolerance: float = 1e-6,
              restart_interval: int = 20):
    """Scalar-Jacobi PCG with the reference's exact recurrence (solver.py:463-508)."""
    if isinstance(equations, NormalEquations):
        dp = equations._live()
        if equations.n_vars == 0:
            return np.zeros(0), PcgResult(0, 0.0)
        it, rel, st = dp.pcg(max_iterations, tolerance, restart_interval)
        if st == _abi.SFB_E_PCG_NONFINITE:
            raise PcgDivergenceError("non-finite values in PCG")
        x = np.zeros(equations.n_vars)
        _abi.check(dp.lib.sfb_get_solution(dp.handle, _abi.ptr(x)), dp.handle)
        return x, PcgResult(it, rel)
    return _pcg_foreign(equations, max_iterations, tolerance, restart_interval)


def _pcg_foreign(equations, max_iterations, tolerance, restart_interval):
    """Duck-typed system (.rhs/.diagonal/.apply): materialise A through the
    caller's own `apply` and run the same device recurrence on it."""
    from .runtime import runtime
    b = np.ascontiguousarray(equations.rhs, dtype=np.float64).reshape(-1)
    n = b.shape[0]
    if n == 0:
        return np.zeros(0), PcgResult(0, 0.0)
    cols = [np.asarray(equations.apply(e), dtype=np.float64).reshape(n) for e in np.eye(n)]
    A = np.ascontiguousarray(np.stack(cols, axis=1))
    diag = np.ascontiguousarray(equations.diagonal, dtype=np.float64).reshape(n)
    rt = runtime()
    x = np.zeros(n)
    import ctypes as C
    it, st = C.c_int32(), C.c_int32()
    rel = C.c_double()
    _abi.check(rt.lib.sfb_pcg_dense(rt.handle, n, _abi.ptr(A), _abi.ptr(b), _abi.ptr(diag),
                                    int(max_iterations), C.c_double(tolerance),
                                    int(restart_interval), _abi.ptr(x), C.byref(it), C.byref(rel),
                                    C.byref(st)), rt.handle)
    if st.value == _abi.SFB_E_PCG_NONFINITE:
        raise PcgDivergenceError("non-finite values in PCG")
    return x, PcgResult(it.value, rel.value)


# ---------------------------------------------------------------------------
# Gauss-Newton driver


@dataclass
class IterationRecord:
    iteration: int
    energy_before: float
    energy_after: float
    dense_weight: float
    pcg_iterations: int
    pcg_residual: float
    step_norm: float
    accepted: bool


@dataclass
class GaussNewtonStats:
    iterations: list = field(default_factory=list)
    converged: bool = False
    aborted: bool = False

    @property
    def final_energy(self):
        return self.iterations[-1].energy_after if self.iterations else 0.0

    def energies_non_increasing(self) -> bool:
        return all(rec.energy_after <= rec.energy_before * (1 + 1e-12) + 1e-15
                   for rec in self.iterations if rec.accepted)


class _EdgeList(list):
    """`dense_edges` as the reference's list of (frame_i, frame_j) tuples, built
    from the device's (n_edges, 2) index array only when first touched (the
    solve loop itself never needs the host copy)."""

    def __init__(self, pairs, frame_ids):
        super().__init__()
        self._pairs = pairs
        self._ids = frame_ids
        self.touched = False

    def _fill(self):
        if not self.touched:
            self.touched = True
            ids = self._ids
            super().extend((ids[a], ids[b]) for a, b in self._pairs.tolist())

    def __len__(self):
        return len(self._pairs) if not self.touched else super().__len__()

    def __bool__(self):
        return len(self) > 0

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __getitem__(self, i):
        self._fill()
        return super().__getitem__(i)

    def __contains__(self, x):
        self._fill()
        return super().__contains__(x)

    def __eq__(self, other):
        self._fill()
        return list.__eq__(self, list(other) if not isinstance(other, list) else other)

    def __ne__(self, other):
        return not self.__eq__(other)

    def __repr__(self):
        self._fill()
        return super().__repr__()

    def __reduce__(self):
        self._fill()
        return (list, (list(super().__iter__()),))

    for _m in ("append", "extend", "insert", "remove", "pop", "clear", "sort", "reverse",
               "__setitem__", "__delitem__", "__iadd__", "index", "count", "copy"):
        def _wrap(name=_m):
            base = getattr(list, name)

            def f(self, *a, **k):
                self._fill()
                return base(self, *a, **k)
            f.__name__ = name
            return f
        locals()[_m] = _wrap()
    del _m, _wrap


class _LazyAssociations(list):
    """Frozen associations of the last linearisation, materialised on first access."""

    def __init__(self, builder):
        super().__init__()
        self._builder = builder
        self._done = False

    def _fill(self):
        if not self._done:
            self._done = True
            super().extend(self._builder())

    def __len__(self):
        self._fill()
        return super().__len__()

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __getitem__(self, i):
        self._fill()
        return super().__getitem__(i)

    def __bool__(self):
        return len(self) > 0


class AlignmentProblem:
    """One joint pose-alignment problem over a set of frames (solver.py:545-750).

    The first frame anchors the gauge.  Dense terms join when `caches` are
    given and the weights ramp them in.  Each instance owns one device
    problem (its own CUDA stream); distinct instances may run concurrently.
    """

    def __init__(self, frame_ids, poses, corr_sets, caches=None, device=None, comm=None):
        self.frame_ids = list(frame_ids)
        if not self.frame_ids:
            raise ValueError("need at least one frame")
        self.poses = {f: poses[f] for f in self.frame_ids}
        self.corr_sets = list(corr_sets)
        self.caches = caches
        self.frame_to_var = {f: k - 1 for k, f in enumerate(self.frame_ids)}
        self.n_vars = 6 * (len(self.frame_ids) - 1)
        for cs in self.corr_sets:  # KeyError for unknown frames, as build_sparse_term
            self.frame_to_var[cs.frame_i], self.frame_to_var[cs.frame_j]
        self._sparse = None
        self.dense_edges = []
        self._device = device
        # data-parallel sharding over frame pairs (paper_1604_01093_b200.shard)
        self._xch = comm if (comm is not None and comm.world > 1) else None
        self._sharded_pcg = self._xch is not None and getattr(comm, "pcg", "replicated") == "sharded"
        self._dp = None
        self._dp_edges = None

    @property
    def sparse(self) -> SparseTerm:
        """Stacked correspondences (solver.py:563); built on first access."""
        if self._sparse is None:
            self._sparse = build_sparse_term(self.corr_sets, self.frame_to_var)
        return self._sparse

    @sparse.setter
    def sparse(self, value):
        self._sparse = value

    # -- device plumbing ---------------------------------------------------
    def _problem(self) -> DeviceProblem:
        if self._dp is None:
            index = {f: k for k, f in enumerate(self.frame_ids)}
            cl = [self.caches[f] for f in self.frame_ids] if self.caches is not None else None
            if cl is not None and len(self.corr_sets) > 256:
                # upload the frames on a helper thread and stack the correspondence
                # sets here as soon as the upload is inside the library (ctypes
                # drops the GIL there), so the two overlap instead of queueing
                rt = runtime(self._device)
                box = {}
                submitted = threading.Event()

                def _upload():
                    try:
                        box["slots"] = rt.slots_for(cl, on_submit=submitted.set)
                    except BaseException as e:  # re-raised on the caller's thread
                        box["e"] = e
                        submitted.set()

                th = threading.Thread(target=_upload, daemon=True)
                th.start()
                submitted.wait()
                dp = None
                try:
                    # the sparse problem is built while the frames are in flight;
                    # the stacked sets live in the runtime's shared pinned staging
                    # until sfb_problem_create has copied them
                    with rt.stage_lock:
                        frames, off, pi, pj = _set_layout(self.corr_sets, index, rt)
                        dp = DeviceProblem(len(self.frame_ids), None, frames, pi, pj, off,
                                           device=self._device)
                finally:
                    th.join()
                try:
                    if "e" in box:
                        raise box["e"]
                    dp.attach_frames(cl, box["slots"])
                except BaseException:
                    dp.close()
                    raise
                self._dp = dp
            else:
                rt = runtime(self._device)
                if cl is not None:
                    rt.slots_for(cl)  # upload outside the staging lock
                with rt.stage_lock:
                    frames, off, pi, pj = _set_layout(self.corr_sets, index, rt)
                    self._dp = DeviceProblem(len(self.frame_ids), cl, frames, pi, pj, off,
                                             device=self._device)
            if self._xch is not None:
                self._dp.set_shard(self._xch.rank, self._xch.world)
                if self._sharded_pcg:
                    self._dp.set_shard_mode(1)
        return self._dp

    def _push_poses(self):
        self._problem().set_poses([self.poses[f] for f in self.frame_ids])

    def _pull_poses(self):
        R, t = self._dp.get_poses()
        host = _host_module()
        if host is not None and type(self.poses) is dict:
            host.make_poses(self.poses, self.frame_ids, R, t, RigidTransform, 1)
            return
        for k, f in enumerate(self.frame_ids[1:], start=1):
            self.poses[f] = RigidTransform(R[k].copy(), t[k].copy())

    def _sync_edges(self):
        if (self.dense_edges is self._dp_edges and isinstance(self.dense_edges, _EdgeList)
                and not self.dense_edges.touched):
            return  # the device already holds exactly these edges
        edges = list(self.dense_edges)
        if edges != self._dp_edges:
            index = {f: k for k, f in enumerate(self.frame_ids)}
            self._dp.set_dense_edges([(index[i], index[j]) for (i, j) in edges])
            self._dp_edges = edges

    def close(self):
        if self._dp is not None:
            self._dp.close()
            self._dp = None

    # -- linearisation ------------------------------------------------------
    def normal_equations(self, weights: EnergyWeights, w_dense: float, config: SolverConfig):
        """(equations, energy, photo_assocs, geo_assocs) at the current poses (solver.py:630-660)."""
        dp = self._problem()
        dp.set_preconditioner(_precond_kind(config))
        self._push_poses()
        self._sync_edges()
        if self._xch is not None and getattr(self._xch, "p2p", False):
            self._xch.p2p_setup(dp)
        e = dp.linearize(weights, w_dense, config, exchange=self._xch)
        dense_on = self.caches is not None and w_dense > 0.0 and bool(self.dense_edges)
        energy = weights.sparse * float(e[0])
        if dense_on:
            energy += w_dense * (weights.photo * float(e[1]) + weights.geo * float(e[2]))
        eqs = NormalEquations(dp, self.n_vars, weights.sparse, self.sparse.var_i, self.sparse.var_j)
        if dense_on:
            directed = _directed_edges(self.dense_edges, config.dense_bidirectional)
            poses = dict(self.poses)
            stride = config.dense_pixel_stride
            photo = _LazyAssociations(lambda: [
                associate_photo(poses, i, j, self.caches[i], self.caches[j], stride)
                for (i, j) in directed] if weights.photo > 0.0 else [])
            geo = _LazyAssociations(lambda: [
                associate_geo(poses, i, j, self.caches[i], self.caches[j], config, stride)
                for (i, j) in directed] if weights.geo > 0.0 else [])
        else:
            photo, geo = [], []
        return eqs, energy, photo, geo

    # -- outer loop ----------------------------------------------------------
    def solve(self, weights: EnergyWeights, config: SolverConfig,
              max_iterations: int = None) -> GaussNewtonStats:
        """Gauss-Newton over the device kernels with the reference's control flow."""
        if max_iterations is None:
            max_iterations = config.batch_iterations
        stats = GaussNewtonStats()
        if self.n_vars == 0:
            stats.converged = True
            return stats
        tr = _Tracer()
        dp = self._problem()
        dp.set_preconditioner(_precond_kind(config))
        self._push_poses()
        tr.mark("setup")
        if self.caches is not None:
            pairs = dp.build_dense_edges(config.view_angle_max_deg, exchange=self._xch)
            self.dense_edges = _EdgeList(pairs, self.frame_ids)
            self._dp_edges = self.dense_edges
        else:
            self._sync_edges()
        if self._xch is not None and getattr(self._xch, "p2p", False):
            self._xch.p2p_setup(dp)  # the structure rebuild may have moved the edge buffer
        have_edges = len(pairs) > 0 if self.caches is not None else bool(self.dense_edges)
        tr.mark("filter")
        if self._sharded_pcg:
            return self._solve_sharded_pcg(dp, weights, config, max_iterations, have_edges, stats, tr)
        best_energy = np.inf
        dp.save_best()
        consecutive_increases = 0
        moved = False
        e_next = None
        for it in range(max_iterations):
            w_dense = dense_ramp_weight(weights, it)
            e = e_next if e_next is not None else dp.linearize(weights, w_dense, config,
                                                               exchange=self._xch)
            e_next = None
            tr.mark("lin")
            dense_on = self.caches is not None and w_dense > 0.0 and have_edges
            energy_before = weights.sparse * float(e[0])
            if dense_on:
                energy_before += w_dense * (weights.photo * float(e[1]) + weights.geo * float(e[2]))
            if energy_before <= 1e-18:
                stats.converged = True
                stats.iterations.append(IterationRecord(
                    it, energy_before, energy_before, w_dense, 0, 0.0, 0.0, True))
                break
            more = it + 1 < max_iterations
            # PCG -> step -> E_after (+ the next linearisation, at the same poses)
            # with one host round trip; the step is skipped on the device when
            # the PCG diverged (PcgDivergenceError -> aborted, solver.py:717-719)
            pcg_it, pcg_rel, diverged, step_norm, ea, e_nx = dp.gn_step(
                weights, w_dense > 0.0, more, dense_ramp_weight(weights, it + 1), config,
                exchange=self._xch)
            if diverged:
                stats.aborted = True
                break
            moved = True
            if more:
                e_next = e_nx
            tr.mark("pcg+step+energy")
            energy_after = weights.sparse * float(ea[0])
            if w_dense > 0.0:
                energy_after += w_dense * (weights.photo * float(ea[1]) + weights.geo * float(ea[2]))
            accepted = energy_after <= energy_before
            stats.iterations.append(IterationRecord(
                it, energy_before, energy_after, w_dense, pcg_it, pcg_rel, step_norm, accepted))
            if accepted:
                consecutive_increases = 0
            else:
                consecutive_increases += 1
                if consecutive_increases >= 2:
                    dp.restore_best()
                    stats.aborted = True
                    break
            if energy_after < best_energy:
                best_energy = energy_after
                dp.save_best()
            if accepted and (energy_before - energy_after) < config.min_relative_decrease * max(
                    energy_before, 1e-30):
                stats.converged = True
                break
        else:
            stats.converged = True
        if moved:
            self._pull_poses()
        tr.mark("pull")
        tr.report()
        return stats


def _solve_sharded_pcg_loop(self, dp, weights, config, max_iterations, have_edges, stats, tr):
    """GN loop of the sharded-PCG mode (ShardComm(pcg="sharded")):
    the reference's control flow (solver.py:681-750) over partial systems -
    one all-reduce per linearisation and frozen-energy pass, one per PCG
    iteration (in sfb_pcg_sharded)."""
    xch = self._xch
    allreduce = xch.pcg_allreduce(dp)
    best_energy = np.inf
    dp.save_best()
    consecutive_increases = 0
    moved = False
    for it in range(max_iterations):
        w_dense = dense_ramp_weight(weights, it)
        e = dp.linearize_sharded(weights, w_dense, config, xch)
        dense_on = self.caches is not None and w_dense > 0.0 and have_edges
        energy_before = weights.sparse * float(e[0])
        if dense_on:
            energy_before += w_dense * (weights.photo * float(e[1]) + weights.geo * float(e[2]))
        if energy_before <= 1e-18:
            stats.converged = True
            stats.iterations.append(IterationRecord(
                it, energy_before, energy_before, w_dense, 0, 0.0, 0.0, True))
            break
        pcg_it, pcg_rel, st = dp.pcg_sharded(config.pcg_max_iterations, config.pcg_tolerance,
                                             config.pcg_restart_interval, allreduce)
        if st == _abi.SFB_E_PCG_NONFINITE:
            stats.aborted = True
            break
        step_norm = dp.apply_step()
        moved = True
        ea = dp.energy_frozen(w_dense > 0.0, exchange=xch)
        tr.mark("pcg+step+energy")
        energy_after = weights.sparse * float(ea[0])
        if w_dense > 0.0:
            energy_after += w_dense * (weights.photo * float(ea[1]) + weights.geo * float(ea[2]))
        accepted = energy_after <= energy_before
        stats.iterations.append(IterationRecord(
            it, energy_before, energy_after, w_dense, pcg_it, pcg_rel, step_norm, accepted))
        if accepted:
            consecutive_increases = 0
        else:
            consecutive_increases += 1
            if consecutive_increases >= 2:
                dp.restore_best()
                stats.aborted = True
                break
        if energy_after < best_energy:
            best_energy = energy_after
            dp.save_best()
        if accepted and (energy_before - energy_after) < config.min_relative_decrease * max(
                energy_before, 1e-30):
            stats.converged = True
            break
    else:
        stats.converged = True
    if moved:
        self._pull_poses()
    tr.mark("pull")
    tr.report()
    return stats


AlignmentProblem._solve_sharded_pcg = _solve_sharded_pcg_loop


class _Tracer:
    """Host wall-time per solve phase, printed to stderr when SFB_TRACE is set."""

    def __init__(self):
        import os
        self.on = bool(os.environ.get("SFB_TRACE"))
        if self.on:
            import time
            self._clock = time.perf_counter
            self.t = self._clock()
            self.acc = {}

    def mark(self, label):
        if self.on:
            now = self._clock()
            self.acc[label] = self.acc.get(label, 0.0) + (now - self.t)
            self.t = now

    def report(self):
        if self.on:
            import sys
            print("sfb trace ms: " + " ".join(f"{k}={1e3 * v:.1f}" for k, v in self.acc.items()),
                  file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# Residual-based pruning


@dataclass
class PruneReport:
    removed_pairs: list
    invalid_frames: list
    rounds: int
    final_max_residual: float


def max_residual_set(poses, corr_sets):
    """Set holding the worst correspondence residual and its value (solver.py:765-776)."""
    worst_set, worst = -1, -1.0
    if not corr_sets:
        return worst_set, worst
    dp = _sparse_problem(poses, corr_sets)
    peaks = dp.sparse_set_max()
    dp.close()
    for idx, cs in enumerate(corr_sets):
        peak = float(peaks[idx]) if len(cs) else 0.0
        if peak > worst:
            worst, worst_set = peak, idx
    return worst_set, worst


def solve_with_pruning(frame_ids, poses, corr_sets, weights, config: SolverConfig,
                       caches=None, max_iterations=None):
    """Alternate solving and pruning of the worst set (solver.py:779-816).

    The device problem stays resident across rounds while the connected
    frames are unchanged: the pruned set's range is emptied on the device
    (sfb_problem_drop_sets; the result equals a problem built without it)
    and the per-set residual maxima of max_residual_set (:765-776) are read
    from the live problem at the solved poses, instead of stacking and
    uploading every set twice per round.  A round that disconnects a frame
    builds a new problem over the remaining frames, as the reference does."""
    sets = list(corr_sets)
    poses = dict(poses)
    removed_pairs, invalid_frames, stats_list = [], [], []
    rounds = 0
    r_max = 0.0
    problem, problem_active = None, None
    try:
        while True:
            rounds += 1
            connected = {f for cs in sets for f in (cs.frame_i, cs.frame_j)}
            active = [f for f in frame_ids if f in connected]
            invalid_frames.extend(f for f in frame_ids if f not in connected and f not in invalid_frames)
            if len(active) < 2 or not sets:
                r_max = 0.0
                break
            if problem is None or active != problem_active:
                if problem is not None:
                    problem.close()
                problem = AlignmentProblem(active, poses, sets, caches)
                problem_active = active
            else:
                problem.poses = {f: poses[f] for f in active}
            stats_list.append(problem.solve(weights, config, max_iterations))
            poses.update(problem.poses)
            peaks = problem._problem().sparse_set_max()
            worst_idx, r_max = -1, -1.0
            for idx, cs in enumerate(sets):
                peak = float(peaks[idx]) if len(cs) else 0.0
                if peak > r_max:
                    r_max, worst_idx = peak, idx
            if r_max <= config.prune_residual_max:
                break
            offender = sets.pop(worst_idx)
            removed_pairs.append((offender.frame_i, offender.frame_j))
            # the device problem compacts its sets the same way (ids follow `sets`)
            problem._problem().drop_sets([worst_idx])
    finally:
        if problem is not None:
            problem.close()
    return poses, sets, PruneReport(removed_pairs, invalid_frames, rounds, r_max), stats_list
