"""Drop-in `scanfuse.tsdf` on B200: the sparse voxel-hashed TSDF volume.

Mirrors the reference module (tsdf.py:1-267): `TsdfVolume(voxel_size,
truncation, depth_weighting)` with `integrate` / `deintegrate(frame,
intrinsics, pose)`, `block`, `allocate`, `blocks`, `block_extent`,
`sorted_coords`, `voxel_state`, `occupied_voxel_count`, plus
`default_truncation`, `volumes_equal`, `save_volume`, `load_volume`,
`VoxelBlock`, `DeintegrationMismatchError`, `BLOCK_SIZE`, `BLOCK_VOXELS`.

The accumulators live on the GPU (libsfb `sfb_tsdf_*`): a frame's truncation
band is sampled into block keys by one kernel, sorted and deduplicated with
CUB, and every touched block is updated by one CTA of 512 voxel threads.
Every voxel decision and every float32 accumulation reproduces the
reference's NumPy arithmetic, so the volume is bit-identical (including the
dict's insertion order and the DeintegrationMismatchError behaviour).

`blocks` and `block()` return host snapshots: mutating their arrays does not
write back (use `allocate` + `load_volume`-style imports to seed data).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._rounding import probe
from .runtime import runtime

BLOCK_SIZE = 8
BLOCK_VOXELS = BLOCK_SIZE ** 3

__all__ = ["BLOCK_SIZE", "BLOCK_VOXELS", "DeintegrationMismatchError", "VoxelBlock", "TsdfVolume",
           "default_truncation", "volumes_equal", "save_volume", "load_volume"]


class DeintegrationMismatchError(RuntimeError):
    """A frame was de-integrated that was never integrated at this pose."""


@dataclass
class VoxelBlock:
    """Accumulators of one 8x8x8 block (flattened to 512), reference tsdf.py:36-52."""

    weight: np.ndarray
    wdist: np.ndarray
    wcolor: np.ndarray

    @classmethod
    def empty(cls):
        return cls(np.zeros(BLOCK_VOXELS, dtype=np.float32), np.zeros(BLOCK_VOXELS, dtype=np.float32),
                   np.zeros((BLOCK_VOXELS, 3), dtype=np.float32))


def default_truncation(voxel_size: float) -> float:
    """tsdf.py:55-57"""
    return max(0.02, 5.0 * voxel_size)


def _f_ordered(a) -> bool:
    a = np.asarray(a)
    return bool(a.flags.f_contiguous and not a.flags.c_contiguous)


class TsdfVolume:
    def __init__(self, voxel_size: float = 0.004, truncation: float = None,
                 depth_weighting: bool = False, device: int | None = None):
        self.voxel_size = float(voxel_size)
        self.truncation = float(truncation if truncation is not None
                                else default_truncation(voxel_size))
        self.depth_weighting = depth_weighting
        self._rt = runtime(device)
        h = C.c_void_p()
        _abi.check(self._rt.lib.sfb_tsdf_create(self._rt.handle, self.voxel_size, self.truncation,
                                                1 if depth_weighting else 0, C.byref(h)),
                   self._rt.handle)
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None:
                self._rt.lib.sfb_tsdf_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # -- hash-grid surface ---------------------------------------------------
    def __len__(self):
        n = C.c_int64()
        _abi.check(self._rt.lib.sfb_tsdf_count(self._h, C.byref(n)), self._h)
        return n.value

    def block(self, coord):
        """Snapshot of the block at `coord`, or None (tsdf.py:70-71)."""
        c = np.asarray([int(x) for x in coord], dtype=np.int64)
        found = C.c_int32()
        b = VoxelBlock.empty()
        _abi.check(self._rt.lib.sfb_tsdf_get_block(self._h, _abi.ptr(c), C.byref(found),
                                                   _abi.ptr(b.weight), _abi.ptr(b.wdist),
                                                   _abi.ptr(b.wcolor)), self._h)
        return b if found.value else None

    def allocate(self, coord) -> VoxelBlock:
        """Existing block, or a new empty one appended to the dict (tsdf.py:73-80)."""
        b = self.block(coord)
        if b is not None:
            return b
        c = np.asarray([[int(x) for x in coord]], dtype=np.int64)
        e = VoxelBlock.empty()
        _abi.check(self._rt.lib.sfb_tsdf_import(self._h, 1, _abi.ptr(c), _abi.ptr(e.weight),
                                                _abi.ptr(e.wdist), _abi.ptr(e.wcolor)), self._h)
        return e

    @property
    def blocks(self) -> dict:
        """{coord: VoxelBlock} in the reference dict's insertion order (a snapshot)."""
        n = len(self)
        coords = np.zeros((n, 3), dtype=np.int64)
        w = np.zeros((n, BLOCK_VOXELS), dtype=np.float32)
        d = np.zeros((n, BLOCK_VOXELS), dtype=np.float32)
        col = np.zeros((n, BLOCK_VOXELS, 3), dtype=np.float32)
        _abi.check(self._rt.lib.sfb_tsdf_export(self._h, n, _abi.ptr(coords), _abi.ptr(w),
                                                _abi.ptr(d), _abi.ptr(col)), self._h)
        return {tuple(int(x) for x in coords[k]): VoxelBlock(w[k], d[k], col[k]) for k in range(n)}

    def _coords(self) -> list:
        n = len(self)
        coords = np.zeros((n, 3), dtype=np.int64)
        _abi.check(self._rt.lib.sfb_tsdf_export(self._h, n, _abi.ptr(coords), None, None, None),
                   self._h)
        return [tuple(int(x) for x in c) for c in coords]

    @property
    def block_extent(self) -> float:
        return self.voxel_size * BLOCK_SIZE

    def sorted_coords(self):
        return sorted(self._coords())

    # -- integration -----------------------------------------------------------
    def integrate(self, frame, intrinsics, pose):
        """Fuse one frame's depth (and color) at the given camera-to-world pose."""
        self._apply(frame, intrinsics, pose, +1)

    def deintegrate(self, frame, intrinsics, pose):
        """Exactly remove a previously integrated frame (same frame, same pose)."""
        self._apply(frame, intrinsics, pose, -1)

    def _apply(self, frame, intrinsics, pose, sign):
        depth = np.ascontiguousarray(frame.depth, dtype=np.float32)
        color = np.ascontiguousarray(frame.color, dtype=np.uint8)
        H, W = depth.shape
        if color.shape != (H, W, 3):
            raise ValueError("colour and depth shapes differ")
        if int(intrinsics.width) != W or int(intrinsics.height) != H:
            # the reference indexes the frame with intrinsics-sized pixel grids
            raise ValueError("intrinsics size does not match the frame")
        pr = probe()
        R = np.asarray(pose.rotation, dtype=np.float64)
        m = int(np.count_nonzero(depth > 0.0))
        f = _f_ordered(pose.rotation)
        pose_ord = (pr["apply_1f"] if f else pr["apply_1"]) if m == 1 else (
            pr["apply_nf"] if f else pr["apply_n"])
        inv = pose.inverse()  # the reference's own inverse, NumPy rounding
        n_s = max(2, int(np.ceil(4.0 * self.truncation / self.block_extent)) + 1)
        tvals = np.ascontiguousarray(np.linspace(0.0, 1.0, n_s), dtype=np.float64)
        k4 = np.array([intrinsics.fx, intrinsics.fy, intrinsics.cx, intrinsics.cy], dtype=np.float64)
        Rp = np.ascontiguousarray(R).reshape(9)
        tp = np.ascontiguousarray(np.asarray(pose.translation, dtype=np.float64)).reshape(3)
        Ri = np.ascontiguousarray(np.asarray(inv.rotation, dtype=np.float64)).reshape(9)
        ti = np.ascontiguousarray(np.asarray(inv.translation, dtype=np.float64)).reshape(3)
        status = C.c_int32()
        ec = np.zeros(3, dtype=np.int64)
        _abi.check(self._rt.lib.sfb_tsdf_apply(
            self._h, sign, W, H, _abi.ptr(color), _abi.ptr(depth), _abi.ptr(k4), _abi.ptr(Rp),
            _abi.ptr(tp), pose_ord, _abi.ptr(Ri), _abi.ptr(ti), pr["apply_n"], _abi.ptr(tvals),
            n_s, C.byref(status), _abi.ptr(ec)), self._h)
        st = status.value
        coord = tuple(int(x) for x in ec)
        if st == 1:
            raise DeintegrationMismatchError("frame has no integrated content")
        if st == 2:
            raise DeintegrationMismatchError(f"block {coord} missing during de-integration")
        if st == 3:
            raise DeintegrationMismatchError(
                f"negative weight in block {coord}: de-integration mismatch")

    # -- read access -----------------------------------------------------------
    def voxel_state(self, world_point):
        """(distance, weight) of the voxel containing a world point; (None, 0) if empty
        (tsdf.py:204-217)."""
        p = np.asarray(world_point, dtype=np.float64)
        voxel = np.floor(p / self.voxel_size).astype(int)
        coord = tuple(np.floor(p / self.block_extent).astype(int))
        block = self.block(coord)
        if block is None:
            return None, 0.0
        local = voxel - np.array(coord) * BLOCK_SIZE
        idx = int(local[0]) * BLOCK_SIZE * BLOCK_SIZE + int(local[1]) * BLOCK_SIZE + int(local[2])
        w = float(block.weight[idx])
        if w <= 0.0:
            return None, 0.0
        return float(block.wdist[idx] / block.weight[idx]), w

    def occupied_voxel_count(self):
        return sum(int(np.count_nonzero(b.weight)) for b in self.blocks.values())

    def _import(self, coords, weight, wdist, wcolor):
        n = len(coords)
        c = np.ascontiguousarray(np.asarray(coords, dtype=np.int64).reshape(n, 3))
        w = np.ascontiguousarray(np.asarray(weight, dtype=np.float32).reshape(n, BLOCK_VOXELS))
        d = np.ascontiguousarray(np.asarray(wdist, dtype=np.float32).reshape(n, BLOCK_VOXELS))
        col = np.ascontiguousarray(np.asarray(wcolor, dtype=np.float32).reshape(n, BLOCK_VOXELS, 3))
        _abi.check(self._rt.lib.sfb_tsdf_import(self._h, n, _abi.ptr(c), _abi.ptr(w), _abi.ptr(d),
                                                _abi.ptr(col)), self._h)


def volumes_equal(a, b, dist_tol: float = 1e-5) -> bool:
    """Equality over occupied voxels: weights exact, distances within tolerance
    (tsdf.py:223-240).  Works on this module's volumes and on reference ones."""
    ba_all, bb_all = a.blocks, b.blocks
    for coord in set(ba_all) | set(bb_all):
        ba, bb = ba_all.get(coord), bb_all.get(coord)
        wa = ba.weight if ba is not None else np.zeros(BLOCK_VOXELS, np.float32)
        wb = bb.weight if bb is not None else np.zeros(BLOCK_VOXELS, np.float32)
        if not np.array_equal(wa, wb):
            return False
        occupied = wa > 0
        if not np.any(occupied):
            continue
        da = ba.wdist[occupied] / wa[occupied]
        db = bb.wdist[occupied] / wb[occupied]
        if np.max(np.abs(da - db)) > dist_tol:
            return False
    return True


def save_volume(path, volume: TsdfVolume):
    """Dump the sparse volume to a .npz archive, sorted block order (tsdf.py:243-257)."""
    blocks = volume.blocks
    coords = sorted(blocks)
    np.savez_compressed(
        path, voxel_size=volume.voxel_size, truncation=volume.truncation,
        coords=np.array(coords, dtype=np.int64).reshape(-1, 3),
        weight=np.stack([blocks[c].weight for c in coords]) if coords
        else np.zeros((0, BLOCK_VOXELS), np.float32),
        wdist=np.stack([blocks[c].wdist for c in coords]) if coords
        else np.zeros((0, BLOCK_VOXELS), np.float32),
        wcolor=np.stack([blocks[c].wcolor for c in coords]) if coords
        else np.zeros((0, BLOCK_VOXELS, 3), np.float32))


def load_volume(path) -> TsdfVolume:
    """tsdf.py:260-267 (blocks inserted in the archive's order)."""
    data = np.load(path)
    volume = TsdfVolume(float(data["voxel_size"]), float(data["truncation"]))
    if data["coords"].shape[0]:
        volume._import(data["coords"], data["weight"], data["wdist"], data["wcolor"])
    return volume
