"""Thin owner of one `sfb_problem` handle (frames + poses + sparse sets on device)."""

from __future__ import annotations

import ctypes as C
import functools
import math

import numpy as np

from . import _abi
from .runtime import runtime


def _pose_arrays(poses: list):
    n = len(poses)
    R = np.empty((n, 3, 3), dtype=np.float64)
    t = np.empty((n, 3), dtype=np.float64)
    fl = np.zeros(n, dtype=np.uint8)
    host = _host_module()
    if host is not None and host.pack_poses(poses, R, t, fl) is not None:
        return R, t, fl
    for k, p in enumerate(poses):
        rot = np.asarray(p.rotation)
        R[k] = rot
        t[k] = np.asarray(p.translation, dtype=np.float64).reshape(3)
        fl[k] = 1 if (rot.flags.f_contiguous and not rot.flags.c_contiguous) else 0
    return R, t, fl


@functools.lru_cache(maxsize=1)
def _host_module():
    """The native host helpers (_sfbhost), or None when not built."""
    try:
        from . import _sfbhost
    except ImportError:
        return None
    return _sfbhost


@functools.lru_cache(maxsize=64)
def view_cos_threshold(max_deg: float) -> float:
    """Smallest c in [-1,1] with degrees(arccos(c)) < max_deg, evaluated with NumPy.

    view_angle_deg (frames.py:183-188) is monotone non-increasing in the
    clipped cosine, so the gate `angle < max_deg` is exactly `c >= c_min`.
    """
    def passes(c: float) -> bool:
        return float(np.degrees(np.arccos(np.clip(c, -1.0, 1.0)))) < max_deg

    if not passes(1.0):
        return math.inf
    if passes(-1.0):
        return -1.0
    lo, hi = -1.0, 1.0  # passes(lo) False, passes(hi) True
    for _ in range(2000):
        mid = 0.5 * (lo + hi)
        if mid == lo or mid == hi:
            break
        if passes(mid):
            hi = mid
        else:
            lo = mid
    # walk to the exact boundary over neighbouring doubles
    while passes(float(np.nextafter(hi, -2.0))) and hi > -1.0:
        hi = float(np.nextafter(hi, -2.0))
    while not passes(hi):
        hi = float(np.nextafter(hi, 2.0))
    return hi


class DeviceProblem:
    """Frames (by cache), poses and correspondence sets resident on one GPU."""

    def __init__(self, n_frames: int, caches_in_order=None, set_frames=None, pts_i=None,
                 pts_j=None, set_offsets=None, device: int | None = None):
        self.rt = runtime(device)
        self.lib = self.rt.lib
        self.n = n_frames
        slots = None
        self._slots = None
        if caches_in_order is not None:
            slots = np.asarray(self.rt.slots_for(caches_in_order), dtype=np.int32)
            self.rt.acquire(slots)
            self._slots = slots
        self._caches = caches_in_order
        if set_frames is None:
            set_frames = np.zeros((0, 2), dtype=np.int32)
        set_frames = np.ascontiguousarray(set_frames, dtype=np.int32).reshape(-1, 2)
        n_sets = set_frames.shape[0]
        fi = np.ascontiguousarray(set_frames[:, 0])
        fj = np.ascontiguousarray(set_frames[:, 1])
        off = np.ascontiguousarray(set_offsets if set_offsets is not None
                                   else np.zeros(n_sets + 1), dtype=np.int64)
        pi = np.ascontiguousarray(pts_i if pts_i is not None else np.zeros((0, 3)), dtype=np.float64)
        pj = np.ascontiguousarray(pts_j if pts_j is not None else np.zeros((0, 3)), dtype=np.float64)
        h = C.c_void_p()
        try:
            _abi.check(self.lib.sfb_problem_create(
                self.rt.handle, n_frames, _abi.ptr(slots), n_sets, _abi.ptr(fi), _abi.ptr(fj),
                _abi.ptr(off), _abi.ptr(pi), _abi.ptr(pj), C.byref(h)), self.rt.handle)
        except BaseException:
            if self._slots is not None:
                self.rt.release_users(self._slots)
                self._slots = None
            raise
        self.handle = h
        self.n_sets = n_sets
        self.n_corr = int(off[-1]) if n_sets else 0
        self.n_vars = 6 * (n_frames - 1)
        self.version = 0

    def attach_frames(self, caches_in_order, slots) -> None:
        """Frames for a problem created without them (uploaded meanwhile)."""
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        self.rt.acquire(slots)
        try:
            self._ck(self.lib.sfb_problem_attach_frames(self.handle, _abi.ptr(slots)))
        except BaseException:
            self.rt.release_users(slots)
            raise
        self._slots = slots
        self._caches = caches_in_order

    def close(self):
        if getattr(self, "handle", None) is not None:
            self.lib.sfb_problem_destroy(self.handle)
            self.handle = None
            if getattr(self, "_slots", None) is not None:
                self.rt.release_users(self._slots)
                self._slots = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc):
        _abi.check(rc, self.handle)

    # -- poses -----------------------------------------------------------------
    def set_poses(self, poses: list) -> None:
        R, t, fl = _pose_arrays(poses)
        self._ck(self.lib.sfb_set_poses(self.handle, _abi.ptr(R), _abi.ptr(t), _abi.ptr(fl)))

    def get_poses(self):
        R = np.empty((self.n, 3, 3))
        t = np.empty((self.n, 3))
        self._ck(self.lib.sfb_get_poses(self.handle, _abi.ptr(R), _abi.ptr(t)))
        return R, t

    def save_best(self):
        self._ck(self.lib.sfb_save_best(self.handle))

    def restore_best(self):
        self._ck(self.lib.sfb_restore_best(self.handle))

    def stream_ptr(self) -> int:
        s = C.c_void_p()
        self._ck(self.lib.sfb_problem_stream(self.handle, C.byref(s)))
        return s.value or 0

    def set_preconditioner(self, kind: int) -> None:
        """0: scalar Jacobi (the reference's), 1: block Jacobi (opt-in)."""
        self._ck(self.lib.sfb_set_preconditioner(self.handle, int(kind)))

    # -- sharding ---------------------------------------
    def set_shard(self, rank: int, world: int) -> None:
        self._ck(self.lib.sfb_set_shard(self.handle, int(rank), int(world)))

    def set_shard_mode(self, mode: int) -> None:
        """0: exchange per-edge sums, replicated PCG; 1: partial systems and the
        sharded PCG (one all-reduce of A.p per iteration)."""
        self._ck(self.lib.sfb_set_shard_mode(self.handle, int(mode)))
        self.shard_mode = int(mode)

    def linearize_sharded(self, weights, w_dense, config, exchange) -> np.ndarray:
        """Sharded-PCG linearisation: this rank's partial system, then one
        all-reduce of [g | Jacobi diagonal | dense energies (| D)]."""
        e = np.zeros(3)
        w, cfg = self._w(weights), self._cfg(config)
        mask = C.c_int32()
        self._ck(self.lib.sfb_linearize_begin(self.handle, C.byref(w), C.c_double(w_dense),
                                              C.byref(cfg), C.byref(mask)))
        self._exchange(exchange, mask.value)
        self._ck(self.lib.sfb_linearize_end_system(self.handle))
        exchange(self, 3)
        self._ck(self.lib.sfb_linearize_finish(self.handle, _abi.ptr(e)))
        self.version += 1
        return e

    def pcg_sharded(self, max_iterations, tolerance, restart_interval, allreduce):
        """PCG over the partial systems; `allreduce(ptr, n, stream)` sums the
        n-double device buffer across ranks in place on `stream`."""
        def cb(_user, ptr, n, stream):
            try:
                allreduce(int(ptr), int(n), int(stream or 0))
                return 0
            except Exception:  # reported as an SfbError by the library
                import traceback
                traceback.print_exc()
                return 1
        fn = _abi.ALLREDUCE_FN(cb)
        it, st = C.c_int32(), C.c_int32()
        rel = C.c_double()
        self._ck(self.lib.sfb_pcg_sharded(self.handle, int(max_iterations), C.c_double(tolerance),
                                          int(restart_interval), fn, None, C.byref(it),
                                          C.byref(rel), C.byref(st)))
        return it.value, rel.value, st.value

    def ipc_export(self, which: int) -> bytes:
        """CUDA IPC handle (64 bytes) of buffer `which` (0 per-edge sums, 1 p2p flags)."""
        h = (C.c_char * 64)()
        nb = C.c_int64()
        self._ck(self.lib.sfb_ipc_export(self.handle, int(which), h, C.byref(nb)))
        return bytes(h)

    def ipc_attach(self, which: int, handles) -> None:
        """Map every rank's buffer `which` (handles indexed by rank)."""
        blob = b"".join(handles)
        buf = C.create_string_buffer(blob, len(blob))
        self._ck(self.lib.sfb_ipc_attach(self.handle, int(which), len(handles), buf))

    def set_p2p(self, on: bool) -> None:
        self._ck(self.lib.sfb_set_p2p(self.handle, 1 if on else 0))

    def exchange_buffer(self, which: int):
        """(device pointer, bytes) of exchange buffer `which` (0 per-edge
        linearisation sums f64, 1 per-edge frozen energies f64, 2 filter
        pass flags u8)."""
        ptr, nb = C.c_void_p(), C.c_int64()
        self._ck(self.lib.sfb_exchange_buffer(self.handle, int(which), C.byref(ptr), C.byref(nb)))
        return ptr.value or 0, nb.value

    shard_mode = 0

    def _exchange(self, exchange, mask: int) -> None:
        for which in (0, 1):
            if mask & (1 << which):
                exchange(self, which)

    # -- pair filter -----------------------------------------------------------
    def build_dense_edges(self, view_angle_max_deg: float, exchange=None) -> np.ndarray:
        n = C.c_int64()
        cos_min = C.c_double(view_cos_threshold(view_angle_max_deg))
        if exchange is None:
            self._ck(self.lib.sfb_build_dense_edges(self.handle, cos_min, C.byref(n)))
        else:
            self._ck(self.lib.sfb_build_dense_edges_begin(self.handle, cos_min))
            exchange(self, 2)
            self._ck(self.lib.sfb_build_dense_edges_end(self.handle, C.byref(n)))
        out = np.zeros((n.value, 2), dtype=np.int32)
        self._ck(self.lib.sfb_get_dense_edges(self.handle, _abi.ptr(out)))
        return out

    def set_dense_edges(self, pairs) -> None:
        arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        self._ck(self.lib.sfb_set_dense_edges(self.handle, arr.shape[0], _abi.ptr(arr)))

    def frustum_overlap(self, pairs) -> np.ndarray:
        arr = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        out = np.zeros(arr.shape[0])
        self._ck(self.lib.sfb_frustum_overlap(self.handle, arr.shape[0], _abi.ptr(arr),
                                              _abi.ptr(out)))
        return out

    # -- GN pieces -------------------------------------------------------------
    @staticmethod
    def _cfg(config):
        return _abi.Config(float(config.geo_distance_max), float(config.geo_normal_min),
                           int(config.dense_pixel_stride), 1 if config.dense_bidirectional else 0)

    @staticmethod
    def _w(weights):
        return _abi.Weights(float(weights.sparse), float(weights.photo), float(weights.geo))

    def linearize(self, weights, w_dense, config, exchange=None) -> np.ndarray:
        e = np.zeros(3)
        w, cfg = self._w(weights), self._cfg(config)
        if exchange is None:
            self._ck(self.lib.sfb_linearize(self.handle, C.byref(w), C.c_double(w_dense),
                                            C.byref(cfg), _abi.ptr(e)))
        else:
            mask = C.c_int32()
            self._ck(self.lib.sfb_linearize_begin(self.handle, C.byref(w), C.c_double(w_dense),
                                                  C.byref(cfg), C.byref(mask)))
            self._exchange(exchange, mask.value)
            self._ck(self.lib.sfb_linearize_end(self.handle, _abi.ptr(e)))
        self.version += 1
        return e

    def energy_and_linearize(self, weights, prev_dense: bool, w_dense_next, config, exchange=None):
        """(frozen energies of the last linearisation, next linearisation energies)
        at the current poses, in one fused device pass."""
        out = np.zeros(6)
        w, cfg = self._w(weights), self._cfg(config)
        pd = 1 if prev_dense else 0
        if exchange is None:
            self._ck(self.lib.sfb_energy_and_linearize(self.handle, C.byref(w), pd,
                                                       C.c_double(w_dense_next), C.byref(cfg),
                                                       _abi.ptr(out)))
        else:
            mask = C.c_int32()
            self._ck(self.lib.sfb_energy_and_linearize_begin(self.handle, C.byref(w), pd,
                                                             C.c_double(w_dense_next),
                                                             C.byref(cfg), C.byref(mask)))
            self._exchange(exchange, mask.value)
            self._ck(self.lib.sfb_energy_and_linearize_end(self.handle, _abi.ptr(out)))
        self.version += 1
        return out[:3], out[3:]

    def pcg(self, max_iterations, tolerance, restart_interval):
        it, st = C.c_int32(), C.c_int32()
        rel = C.c_double()
        self._ck(self.lib.sfb_pcg(self.handle, int(max_iterations), C.c_double(tolerance),
                                  int(restart_interval), C.byref(it), C.byref(rel), C.byref(st)))
        return it.value, rel.value, st.value

    def apply_step(self) -> float:
        s = C.c_double()
        self._ck(self.lib.sfb_apply_step(self.handle, C.byref(s)))
        return s.value

    def energy_frozen(self, dense: bool, exchange=None) -> np.ndarray:
        e = np.zeros(3)
        if exchange is None:
            self._ck(self.lib.sfb_energy_frozen(self.handle, 1 if dense else 0, _abi.ptr(e)))
        else:
            mask = C.c_int32()
            self._ck(self.lib.sfb_energy_frozen_begin(self.handle, 1 if dense else 0,
                                                      C.byref(mask)))
            self._exchange(exchange, mask.value)
            self._ck(self.lib.sfb_energy_frozen_end(self.handle, _abi.ptr(e)))
        return e

    def gn_step(self, weights, prev_dense: bool, relinearize: bool, w_dense_next, config,
                exchange=None):
        """PCG -> step -> frozen energy (+ next linearisation) in one round trip.
        Returns (pcg_it, pcg_rel, diverged, step_norm, e_after[3], e_next[3])."""
        out = np.zeros(10)
        w, cfg = self._w(weights), self._cfg(config)
        args = (self.handle, int(config.pcg_max_iterations), C.c_double(config.pcg_tolerance),
                int(config.pcg_restart_interval), C.byref(w), 1 if prev_dense else 0,
                1 if relinearize else 0, C.c_double(w_dense_next), C.byref(cfg))
        if exchange is None:
            self._ck(self.lib.sfb_gn_step(*args, _abi.ptr(out)))
        else:
            mask = C.c_int32()
            self._ck(self.lib.sfb_gn_step_begin(*args, C.byref(mask)))
            self._exchange(exchange, mask.value)
            self._ck(self.lib.sfb_gn_step_end(self.handle, _abi.ptr(out)))
        if relinearize:
            self.version += 1
        return int(out[0]), float(out[1]), bool(out[2]), float(out[3]), out[4:7], out[7:10]

    def gn_iteration(self, weights, w_dense, config):
        w, cfg = self._w(weights), self._cfg(config)
        out = _abi.IterResult()
        self._ck(self.lib.sfb_gn_iteration(
            self.handle, C.byref(w), C.c_double(w_dense), C.byref(cfg),
            int(config.pcg_max_iterations), C.c_double(config.pcg_tolerance),
            int(config.pcg_restart_interval), C.byref(out)))
        self.version += 1
        return out

    # -- measurement -----------------------------------------------------------
    def profile(self, enable: bool = True) -> None:
        self._ck(self.lib.sfb_profile(self.handle, 1 if enable else 0))

    def profile_read(self, reset: bool = True) -> dict:
        ms = np.zeros(8)
        n = np.zeros(8, dtype=np.int64)
        self._ck(self.lib.sfb_profile_read(self.handle, _abi.ptr(ms), _abi.ptr(n), 1 if reset else 0))
        return {name: (float(ms[k]), int(n[k])) for k, name in enumerate(_abi.PROF_CLASSES)}

    # -- host views ------------------------------------------------------------
    def dims(self):
        nv, npairs, nc = C.c_int32(), C.c_int64(), C.c_int64()
        self._ck(self.lib.sfb_system_dims(self.handle, C.byref(nv), C.byref(npairs), C.byref(nc)))
        return nv.value, npairs.value, nc.value

    def matvec(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(self.n_vars)
        y = np.zeros(self.n_vars)
        self._ck(self.lib.sfb_matvec(self.handle, _abi.ptr(x), _abi.ptr(y)))
        return y

    def gradient(self) -> np.ndarray:
        g = np.zeros(self.n_vars)
        self._ck(self.lib.sfb_get_gradient(self.handle, _abi.ptr(g)))
        return g

    def diagonal(self) -> np.ndarray:
        d = np.zeros(self.n_vars)
        self._ck(self.lib.sfb_get_diagonal(self.handle, _abi.ptr(d)))
        return d

    def blocks(self):
        nv, npairs, _ = self.dims()
        D = np.zeros((nv // 6, 6, 6))
        B = np.zeros((npairs, 6, 6))
        pv = np.zeros((npairs, 2), dtype=np.int32)
        self._ck(self.lib.sfb_get_blocks(self.handle, _abi.ptr(D), _abi.ptr(B), _abi.ptr(pv)))
        return D, B, pv

    def sparse_world(self):
        wi = np.zeros((self.n_corr, 3))
        wj = np.zeros((self.n_corr, 3))
        if self.n_corr:
            self._ck(self.lib.sfb_get_sparse_world(self.handle, _abi.ptr(wi), _abi.ptr(wj)))
        return wi, wj

    def sparse_residuals(self) -> np.ndarray:
        r = np.zeros((self.n_corr, 3))
        if self.n_corr:
            self._ck(self.lib.sfb_sparse_residuals(self.handle, _abi.ptr(r)))
        return r

    def drop_sets(self, set_ids) -> None:
        """Empty the given correspondence sets on the device (sfb_problem_drop_sets)."""
        ids = np.ascontiguousarray(set_ids, dtype=np.int32)
        self._ck(self.lib.sfb_problem_drop_sets(self.handle, int(ids.size), _abi.ptr(ids)))

    def sparse_set_max(self) -> np.ndarray:
        m = np.zeros(self.n_sets)
        if self.n_sets:
            self._ck(self.lib.sfb_sparse_set_max(self.handle, _abi.ptr(m)))
        return m

    def associate(self, fi: int, fj: int, kind: int, config):
        cfg = self._cfg(config)
        c = self._caches[fi]
        hw = np.asarray(c.valid_depth).size
        sel = np.zeros(hw, dtype=np.uint8)
        tgt = np.zeros(hw, dtype=np.int32)
        self._ck(self.lib.sfb_associate(self.handle, fi, fj, kind, C.byref(cfg), _abi.ptr(sel),
                                        _abi.ptr(tgt)))
        return sel.astype(bool), tgt

    def point_eval(self, fi, fj, kind, points, aux, targets=None, jacobian=True):
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        m = pts.shape[0]
        aux = np.ascontiguousarray(aux, dtype=np.float64)
        tg = None if targets is None else np.ascontiguousarray(targets, dtype=np.float64)
        res = np.zeros((m, 2) if kind == 0 else (m,))
        jac = (np.zeros((m, 2, 6) if kind == 0 else (m, 6))) if jacobian else None
        self._ck(self.lib.sfb_point_eval(self.handle, fi, fj, kind, m, _abi.ptr(pts),
                                         _abi.ptr(aux), _abi.ptr(tg), _abi.ptr(res),
                                         _abi.ptr(jac)))
        return res, jac
