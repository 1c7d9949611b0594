"""Device runtime: one libsfb context per CUDA device plus its frame store.

A `CachedFrame` is immutable after construction (reference frames.py:8-9),
so its planes are uploaded once per context and addressed by slot.  The
store keys frames by object identity and holds only a weak reference: when
the caller drops a cache, its slot (and device block) is released as soon
as no live device problem still uses it.  Problems register the slots they
read (`acquire` / `release_users`); `clear_frames()` forgets every mapping
and releases the slots nobody uses, deferring the rest to the last user.
Caches that cannot be weakly referenced are held strongly until
`clear_frames()`.
"""

from __future__ import annotations

import ctypes as C
import os
import contextlib
import threading
import weakref

import numpy as np

from . import _abi
from ._rounding import probe


def _default_device() -> int:
    for key in ("SFB_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0


def _plane(a, dtype, shape) -> np.ndarray:
    if isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous:
        arr = a  # fast path: already the layout the library reads
    else:
        arr = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    if arr.shape != shape:
        raise ValueError(f"cache plane has shape {arr.shape}, expected {shape}")
    return arr


# numpy twin of sfb_frame_desc (include/sfb.h), so 500 descriptors fill by column
_DESC_DTYPE = np.dtype([("width", "<i4"), ("height", "<i4"), ("fx", "<f8"), ("fy", "<f8"),
                        ("cx", "<f8"), ("cy", "<f8"), ("valid_depth", "<u8"),
                        ("valid_normal", "<u8"), ("points", "<u8"), ("normals", "<u8"),
                        ("grad", "<u8")], align=True)


def _addr(a: np.ndarray) -> int:
    """Data pointer of a C-contiguous array (ctypes.c_char.from_buffer is ~2x
    cheaper than ndarray.ctypes.data; read-only buffers fall back)."""
    try:
        return C.addressof(C.c_char.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data


class Runtime:
    def __init__(self, device: int):
        self.lib = _abi.load()
        self.device = device
        h = C.c_void_p()
        _abi.check(self.lib.sfb_ctx_create(device, C.byref(h)))
        self.handle = h
        pr = probe()
        r = _abi.Rounding(**{k: pr[k] for k, _ in _abi.Rounding._fields_})
        _abi.check(self.lib.sfb_ctx_set_rounding(h, C.byref(r)), h)
        # id(cache) -> (slot, weakref to the cache, or the cache itself)
        self._frames: dict[int, tuple[int, object]] = {}
        self._with_intensity: set[int] = set()  # slots holding intensity_low
        self._users: dict[int, int] = {}        # slot -> live users (problems, calls)
        self._orphans: set[int] = set()         # unmapped slots waiting for their last user
        self._dead: list = []                   # ids of collected caches (weakref callbacks append)
        self._staging: dict = {}
        self._staging_addr: dict = {}
        self._staging_ptrs: list = []
        # RLock: a cache's weakref callback never takes it (it only appends to _dead),
        # but slot bookkeeping may be re-entered from one call chain
        self._lock = threading.RLock()
        # held from stacking correspondence sets into the shared pinned
        # staging until sfb_problem_create has copied them
        self.stage_lock = threading.Lock()

    # -- frame store --------------------------------------------------------
    def slots_for(self, caches, on_submit=None) -> list[int]:
        """Slots of the given caches, uploading the ones not yet resident.
        `on_submit()` runs once the upload is about to enter the library (which
        drops the GIL), or right away when nothing needs uploading."""
        try:
            with self._lock:
                self._reap()
                missing = []
                seen = set()
                for c in caches:
                    if self._lookup(c) is None and id(c) not in seen:
                        missing.append(c)
                        seen.add(id(c))
                if missing:
                    self._upload(missing, on_submit)
                    on_submit = None
                return [self._frames[id(c)][0] for c in caches]
        finally:
            if on_submit is not None:
                on_submit()

    def _upload(self, caches, on_submit=None) -> None:
        n = len(caches)
        descs = np.zeros(n, dtype=_DESC_DTYPE)  # the sfb_frame_desc array
        try:
            from . import _sfbhost
            native = _sfbhost.fill_frame_descs(caches, descs) is not None
        except ImportError:
            native = False
        if native:  # every plane already in the library's layout: no copies
            slots = np.zeros(n, dtype=np.int32)
            if on_submit is not None:
                on_submit()
            _abi.check(self.lib.sfb_frames_upload(self.handle, n, descs.ctypes.data_as(
                C.POINTER(_abi.FrameDesc)), _abi.ptr(slots)), self.handle)
            for c, s in zip(caches, slots):
                self._register(c, int(s))
            return
        keep = []
        dims = np.empty((n, 2), dtype=np.int32)
        kk = np.empty((n, 4), dtype=np.float64)
        ptrs = np.empty((n, 5), dtype=np.uint64)
        for k, c in enumerate(caches):
            vd = c.valid_depth
            h, w = np.shape(vd)
            planes = (
                _plane(vd, np.bool_, (h, w)).view(np.uint8),
                _plane(c.valid_normal, np.bool_, (h, w)).view(np.uint8),
                _plane(c.points_low, np.float32, (h, w, 3)),
                _plane(c.normals_low, np.float32, (h, w, 3)),
                _plane(c.grad_low, np.float32, (h, w, 2)),
            )
            keep.append(planes)
            k_low = c.intrinsics_low
            if int(k_low.width) != w or int(k_low.height) != h:
                raise ValueError("intrinsics_low size does not match the cache planes")
            dims[k] = (w, h)
            kk[k] = (k_low.fx, k_low.fy, k_low.cx, k_low.cy)
            ptrs[k] = [_addr(p) for p in planes]
        descs["width"], descs["height"] = dims[:, 0], dims[:, 1]
        for q, name in enumerate(("fx", "fy", "cx", "cy")):
            descs[name] = kk[:, q]
        for q, name in enumerate(("valid_depth", "valid_normal", "points", "normals", "grad")):
            descs[name] = ptrs[:, q]
        slots = np.zeros(n, dtype=np.int32)
        if on_submit is not None:
            on_submit()
        _abi.check(self.lib.sfb_frames_upload(self.handle, n, descs.ctypes.data_as(
            C.POINTER(_abi.FrameDesc)), _abi.ptr(slots)), self.handle)
        for c, s in zip(caches, slots):
            self._register(c, int(s))
        del keep

    def intensity_slots_for(self, caches) -> list[int]:
        """Slots of the caches with their intensity_low plane resident as well
        (dense_verify's colour gate; the solver path never uploads it)."""
        slots = self.slots_for(caches)
        with self._lock:
            todo, keep, seen = [], [], set()
            for c, s in zip(caches, slots):
                if s in self._with_intensity or s in seen:
                    continue
                h, w = np.asarray(c.valid_depth).shape
                keep.append(_plane(c.intensity_low, np.float32, (h, w)))
                todo.append(s)
                seen.add(s)
            if todo:
                arr = np.asarray(todo, dtype=np.int32)
                ptrs = (C.c_void_p * len(todo))(*[k.ctypes.data for k in keep])
                _abi.check(self.lib.sfb_frames_set_intensity(self.handle, len(todo), _abi.ptr(arr),
                                                             ptrs), self.handle)
                self._with_intensity.update(todo)
        return slots

    def staging(self, key: str, nbytes: int) -> np.ndarray:
        """A reusable page-locked host byte buffer of at least nbytes (grown
        geometrically); its contents are clobbered by the next caller of the
        same key, so users consume it before returning."""
        buf = self._staging.get(key)
        if buf is None or buf.nbytes < nbytes:
            size = max(int(nbytes), 2 * (buf.nbytes if buf is not None else 0), 1 << 16)
            ptr = C.c_void_p()
            _abi.check(self.lib.sfb_host_alloc(size, C.byref(ptr)))
            arr = np.ctypeslib.as_array((C.c_uint8 * size).from_address(ptr.value))
            if buf is not None:
                self._staging_ptrs.append(self._staging_addr[key])  # freed with the runtime
            self._staging[key] = arr
            self._staging_addr[key] = ptr.value
            buf = arr
        return buf

    def adopt(self, caches, slots) -> None:
        """Register caches whose planes were produced on the device
        (sfb_build_cache): already resident, intensity included."""
        with self._lock:
            self._reap()
            for c, s in zip(caches, slots):
                self._register(c, int(s))
                self._with_intensity.add(int(s))

    # -- slot lifetime ----------------------------------------------------------
    def _register(self, cache, slot: int) -> None:
        try:
            # a callback weakref (~1 us) rather than weakref.finalize (~2.5 us,
            # 5 ms per 2,000-frame upload): the entry keeps the ref alive, so
            # the callback fires exactly while the cache is mapped
            ref = weakref.ref(cache, lambda _r, k=id(cache), dead=self._dead: dead.append(k))
        except TypeError:  # not weakly referenceable: held until clear_frames()
            ref = cache
        self._frames[id(cache)] = (slot, ref)

    def _lookup(self, cache):
        ent = self._frames.get(id(cache))
        if ent is None:
            return None
        ref = ent[1]
        alive = ref() if isinstance(ref, weakref.ref) else ref
        if alive is not cache:  # a recycled id: the old cache is gone
            self._forget(id(cache))
            return None
        return ent[0]

    def _forget(self, key) -> None:
        ent = self._frames.pop(key, None)
        if ent is not None:
            self._orphans.add(ent[0])

    def _reap(self) -> None:
        """Unmap collected caches; release unmapped slots nobody uses."""
        while self._dead:
            key = self._dead.pop()
            ent = self._frames.get(key)
            if ent is not None and isinstance(ent[1], weakref.ref) and ent[1]() is None:
                self._forget(key)
        free = [s for s in self._orphans if self._users.get(s, 0) == 0]
        if free:
            arr = np.array(sorted(free), dtype=np.int32)
            _abi.check(self.lib.sfb_frames_release(self.handle, len(arr), _abi.ptr(arr)),
                       self.handle)
            self._orphans.difference_update(free)
            self._with_intensity.difference_update(free)

    def acquire(self, slots) -> None:
        """Register a user (a device problem) of these slots."""
        with self._lock:
            for s in set(int(x) for x in slots):
                self._users[s] = self._users.get(s, 0) + 1

    def release_users(self, slots) -> None:
        with self._lock:
            for s in set(int(x) for x in slots):
                n = self._users.get(s, 0) - 1
                if n <= 0:
                    self._users.pop(s, None)
                else:
                    self._users[s] = n
            self._reap()

    @contextlib.contextmanager
    def using(self, slots):
        """Keep the slots alive for the duration of one library call."""
        self.acquire(slots)
        try:
            yield
        finally:
            self.release_users(slots)

    def resident_frames(self) -> int:
        """Slots currently held (mapped or awaiting their last user)."""
        with self._lock:
            self._reap()
            return len(self._frames) + len(self._orphans)

    def clear_frames(self) -> None:
        """Forget every cache mapping; slots still used by live problems are
        released when their last user closes."""
        with self._lock:
            for key in list(self._frames):
                self._forget(key)
            self._reap()

    def __del__(self):
        try:
            for ptr in list(self._staging_addr.values()) + self._staging_ptrs:
                self.lib.sfb_host_free(C.c_void_p(ptr))
            self.lib.sfb_ctx_destroy(self.handle)
        except Exception:
            pass


_runtimes: dict[int, Runtime] = {}
_rt_lock = threading.Lock()


def runtime(device: int | None = None) -> Runtime:
    dev = _default_device() if device is None else int(device)
    with _rt_lock:
        rt = _runtimes.get(dev)
        if rt is None:
            rt = Runtime(dev)
            _runtimes[dev] = rt
        return rt
