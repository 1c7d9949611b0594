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

`blocks` is a live mapping view of the device volume, in the reference
dict's insertion order: `blocks[coord]` fetches one block (cached until the
next integrate / deintegrate / assignment), `blocks[coord] = VoxelBlock(...)`
writes through to the device (how the reference's `load_volume` seeds a
volume, tsdf.py:260-267), iteration yields coordinates, and `items()` /
`values()` export the whole volume once.  Blocks handed out (`blocks[c]`,
`block()`, `allocate()`) are read-only host copies: writing into their
arrays raises instead of being silently lost.
"""

from __future__ import annotations

import ctypes as C
from collections.abc import MutableMapping
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._rounding import probe
from .runtime import runtime

BLOCK_SIZE = 8
BLOCK_VOXELS = BLOCK_SIZE ** 3

__all__ = ["BLOCK_SIZE", "BLOCK_VOXELS", "DeintegrationMismatchError", "VoxelBlock", "TsdfVolume",
           "BlockView",
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

    def _key(self, coord) -> tuple:
        return tuple(int(x) for x in coord)

    def _fetch(self, key):
        """One block from the device (read-only host copy), or None."""
        c = np.asarray(key, dtype=np.int64)
        found = C.c_int32()
        b = VoxelBlock.empty()
        _abi.check(self._rt.lib.sfb_tsdf_get_block(self._h, _abi.ptr(c), C.byref(found),
                                                   _abi.ptr(b.weight), _abi.ptr(b.wdist),
                                                   _abi.ptr(b.wcolor)), self._h)
        return _readonly(b) if found.value else None

    def block(self, coord):
        """The block at `coord`, or None (tsdf.py:70-71)."""
        return self.blocks.get(self._key(coord))

    def allocate(self, coord) -> VoxelBlock:
        """Existing block, or a new empty one appended to the dict (tsdf.py:73-80)."""
        key = self._key(coord)
        b = self.blocks.get(key)
        if b is not None:
            return b
        self.blocks[key] = VoxelBlock.empty()
        return self.blocks[key]

    @property
    def blocks(self) -> "BlockView":
        """{coord: VoxelBlock} view in the reference dict's insertion order."""
        view = getattr(self, "_view", None)
        if view is None:
            view = self._view = BlockView(self)
        return view

    def snapshot(self) -> dict:
        """Every block at once, {coord: VoxelBlock} (one export)."""
        n = len(self)
        coords = np.zeros((n, 3), dtype=np.int64)
        w = np.zeros((n, BLOCK_VOXELS), dtype=np.float32)
        d = np.zeros((n, BLOCK_VOXELS), dtype=np.float32)
        col = np.zeros((n, BLOCK_VOXELS, 3), dtype=np.float32)
        _abi.check(self._rt.lib.sfb_tsdf_export(self._h, n, _abi.ptr(coords), _abi.ptr(w),
                                                _abi.ptr(d), _abi.ptr(col)), self._h)
        for a in (w, d, col):
            a.flags.writeable = False
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
        self._version = getattr(self, "_version", 0) + 1
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
        self._version = getattr(self, "_version", 0) + 1
        n = len(coords)
        c = np.ascontiguousarray(np.asarray(coords, dtype=np.int64).reshape(n, 3))
        w = np.ascontiguousarray(np.asarray(weight, dtype=np.float32).reshape(n, BLOCK_VOXELS))
        d = np.ascontiguousarray(np.asarray(wdist, dtype=np.float32).reshape(n, BLOCK_VOXELS))
        col = np.ascontiguousarray(np.asarray(wcolor, dtype=np.float32).reshape(n, BLOCK_VOXELS, 3))
        _abi.check(self._rt.lib.sfb_tsdf_import(self._h, n, _abi.ptr(c), _abi.ptr(w), _abi.ptr(d),
                                                _abi.ptr(col)), self._h)


def _readonly(b: VoxelBlock) -> VoxelBlock:
    for a in (b.weight, b.wdist, b.wcolor):
        a.flags.writeable = False
    return b


class BlockView(MutableMapping):
    """Live {coord: VoxelBlock} view of a device TsdfVolume (the reference's
    `TsdfVolume.blocks` dict, tsdf.py:65)."""

    def __init__(self, volume: TsdfVolume):
        self._vol = volume
        self._ver = None
        self._cache = {}
        self._order = None

    def _fresh(self):
        ver = getattr(self._vol, "_version", 0)
        if ver != self._ver:
            self._ver = ver
            self._cache.clear()
            self._order = None

    def __getitem__(self, coord):
        key = self._vol._key(coord)
        self._fresh()
        b = self._cache.get(key)
        if b is None:
            b = self._vol._fetch(key)
            if b is None:
                raise KeyError(key)
            self._cache[key] = b
        return b

    def __setitem__(self, coord, block):
        """Write one block through to the device (new keys append, as a dict)."""
        self._vol._import([self._vol._key(coord)], [block.weight], [block.wdist], [block.wcolor])

    def __delitem__(self, coord):
        raise TypeError("device TsdfVolume blocks are removed by deintegrate() only")

    def __iter__(self):
        self._fresh()
        if self._order is None:
            self._order = self._vol._coords()
        return iter(list(self._order))

    def __len__(self):
        return len(self._vol)

    def __contains__(self, coord):
        try:
            self[coord]
        except KeyError:
            return False
        return True

    def _all(self) -> dict:
        self._fresh()
        snap = self._vol.snapshot()
        self._cache.update(snap)
        self._order = list(snap)
        return snap

    def items(self):
        return self._all().items()

    def values(self):
        return self._all().values()

    def copy(self) -> dict:
        return dict(self._all())

    def __repr__(self):
        return f"<TsdfVolume.blocks: {len(self)} blocks>"


def _blocks_dict(volume) -> dict:
    """All blocks of a device volume (one export) or a reference volume's dict."""
    if isinstance(volume, TsdfVolume):
        return volume.snapshot()
    return volume.blocks


def volumes_equal(a, b, dist_tol: float = 1e-5) -> bool:
    """Equality over occupied voxels: weights exact, distances within tolerance
    (tsdf.py:223-240).  Works on this module's volumes and on reference ones."""
    ba_all, bb_all = _blocks_dict(a), _blocks_dict(b)
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
    blocks = _blocks_dict(volume)
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
    if data["coords"].shape[0]:  # one batched write (the reference assigns block by block)
        volume._import(data["coords"], data["weight"], data["wdist"], data["wcolor"])
    return volume
