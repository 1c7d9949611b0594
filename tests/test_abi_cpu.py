"""CPU-only checks of the boundary: the library loads, exports every symbol the
header declares, the ctypes table matches the header, and host-side helpers
(rounding probe, angle threshold, synthetic inputs) behave."""

import ctypes
import math
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sfb.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sfb_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1604_01093_b200 import _build
    _build.build()
    from paper_1604_01093_b200 import _abi
    return _abi.load()


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_1604_01093_b200" / "libsfb.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (sfb_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_ctypes_table_covers_header(lib):
    from paper_1604_01093_b200 import _abi
    declared = set(_abi.SIGNATURES) | {"sfb_last_error", "sfb_abi_version"}
    assert set(header_symbols()) == declared


def test_abi_version_and_no_device_error(lib):
    from paper_1604_01093_b200 import _abi
    assert lib.sfb_abi_version() == 1
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        h = ctypes.c_void_p()
        rc = lib.sfb_ctx_create(0, ctypes.byref(h))
        assert rc == _abi.SFB_E_CUDA
        assert b"CUDA" in lib.sfb_last_error(None) or lib.sfb_last_error(None)


def test_sm100a_cubin_present():
    so = ROOT / "paper_1604_01093_b200" / "libsfb.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_rounding_probe_matches_numpy():
    from paper_1604_01093_b200._rounding import PERMS, chain, probe
    codes = probe()
    rng = np.random.default_rng(5)
    for _ in range(200):
        a, b = rng.normal(size=3), rng.normal(size=3)
        assert chain(a, b, codes["dot3"]) == float(np.dot(a, b))
        M = rng.normal(size=(3, 3))
        M[0] = a
        assert chain(a, b, codes["matvec_c"]) == float((M @ b)[0])
    assert len(PERMS) == 6


@pytest.mark.parametrize("deg", [60.0, 30.0, 45.0, 89.9, 0.5, 180.0, 200.0, 0.0])
def test_view_cos_threshold_is_exact_preimage(deg):
    from paper_1604_01093_b200.device_problem import view_cos_threshold
    c = view_cos_threshold(deg)

    def passes(x):
        return float(np.degrees(np.arccos(np.clip(x, -1.0, 1.0)))) < deg

    if math.isinf(c):
        assert not passes(1.0)
        return
    assert passes(c)
    below = float(np.nextafter(c, -2.0))
    assert c == -1.0 or not passes(below)
    rng = np.random.default_rng(0)
    for x in np.concatenate([rng.uniform(-1, 1, 500), c + np.arange(-50, 50) * 1e-16]):
        assert passes(x) == (np.clip(x, -1, 1) >= c)


def test_synth_deterministic():
    from scenes import synth
    a, b = synth.make("cfg2"), synth.make("cfg2")
    assert synth.cache_digest(a.caches) == synth.cache_digest(b.caches)
    assert all(np.array_equal(x.points_i, y.points_i) for x, y in zip(a.corr_sets, b.corr_sets))


def test_build_cache_matches_reference_fixture():
    from golden_io import GoldenScene
    s = GoldenScene("cfg2")
    assert s.cache_sha_ok


def test_native_set_stacking_matches_numpy_path():
    """_sfbhost.stack_sets_into == the NumPy stacking (build_sparse_term order),
    falls back (None) on non-float64 points, and raises like the reference."""
    import copy
    from paper_1604_01093_b200 import _build
    _build.build_host()
    from paper_1604_01093_b200 import _sfbhost
    from scenes import synth
    from paper_1604_01093_b200 import solver as S
    sc = synth.make("cfg3")
    index = {f: k for k, f in enumerate(sc.frame_ids)}
    sets = sc.corr_sets
    n = len(sets)
    fr = np.empty(2 * n, np.int32)
    of = np.empty(n + 1, np.int64)
    small = np.empty(3, np.float64)
    need = _sfbhost.stack_sets_into(sets, index, fr, of, small, small)
    rows = -need - 1
    assert rows == sum(len(s) for s in sets)
    pi = np.empty(3 * rows)
    pj = np.empty(3 * rows)
    assert _sfbhost.stack_sets_into(sets, index, fr, of, pi, pj) == rows
    ref = S._set_layout(sets, index)
    assert np.array_equal(fr.reshape(-1, 2), ref[0]) and np.array_equal(of, ref[1])
    assert np.array_equal(pi.reshape(-1, 3), ref[2]) and np.array_equal(pj.reshape(-1, 3), ref[3])
    odd = copy.copy(sets[3])
    odd.points_i = odd.points_i.astype(np.float32)
    assert _sfbhost.stack_sets_into([sets[0], odd], index, fr, of, pi, pj) is None
    bad = copy.copy(sets[1])
    bad.frame_j = 10 ** 7
    with pytest.raises(KeyError):
        _sfbhost.stack_sets_into([bad], index, fr, of, pi, pj)
    short = copy.copy(sets[2])
    short.points_j = short.points_j[:-1]
    with pytest.raises(ValueError):
        _sfbhost.stack_sets_into([short], index, fr, of, pi, pj)


def test_native_frame_descriptors():
    from paper_1604_01093_b200 import _build
    _build.build_host()
    from paper_1604_01093_b200 import _sfbhost
    from scenes import synth
    from paper_1604_01093_b200.runtime import _DESC_DTYPE
    sc = synth.make("cfg2")
    caches = [sc.caches[f] for f in sc.frame_ids]
    d = np.zeros(len(caches), dtype=_DESC_DTYPE)
    assert _sfbhost.fill_frame_descs(caches, d) is True
    for k, c in enumerate(caches):
        assert (d[k]["width"], d[k]["height"]) == c.valid_depth.shape[::-1]
        assert d[k]["points"] == c.points_low.ctypes.data
        assert d[k]["grad"] == c.grad_low.ctypes.data
        assert d[k]["fx"] == c.intrinsics_low.fx and d[k]["cy"] == c.intrinsics_low.cy
    import copy
    odd = copy.copy(caches[0])
    odd.points_low = np.asfortranarray(odd.points_low)
    assert _sfbhost.fill_frame_descs([odd], d) is None


def _py_pose_arrays(poses):
    """device_problem._pose_arrays' NumPy loop, restated as the checker."""
    n = len(poses)
    R, t, fl = np.empty((n, 3, 3)), np.empty((n, 3)), np.zeros(n, np.uint8)
    for k, p in enumerate(poses):
        rot = np.asarray(p.rotation)
        R[k] = rot
        t[k] = np.asarray(p.translation, dtype=np.float64).reshape(3)
        fl[k] = 1 if (rot.flags.f_contiguous and not rot.flags.c_contiguous) else 0
    return R, t, fl


def test_native_pose_packing_matches_numpy_path():
    """_sfbhost.pack_poses / make_poses == the NumPy pose push / pull, including
    F-ordered and strided rotations (the BLAS-order flag) and the fallback."""
    from paper_1604_01093_b200 import _build
    _build.build_host()
    from paper_1604_01093_b200 import _sfbhost
    from paper_1604_01093_b200.device_problem import _pose_arrays
    from paper_1604_01093_b200.solver import RigidTransform
    rng = np.random.default_rng(3)
    poses = [RigidTransform(rng.standard_normal((3, 3)), rng.standard_normal(3)) for _ in range(40)]
    poses[2] = RigidTransform(np.asfortranarray(poses[2].rotation), poses[2].translation.reshape(3, 1).copy())
    poses[3] = RigidTransform(rng.standard_normal((3, 5))[:, 1:4], rng.standard_normal((3, 2))[:, 1])
    n = len(poses)
    R, t, fl = np.empty((n, 3, 3)), np.empty((n, 3)), np.zeros(n, np.uint8)
    assert _sfbhost.pack_poses(poses, R, t, fl) is True
    for got, want in zip((R, t, fl), _py_pose_arrays(poses)):
        assert np.array_equal(got, want)
    assert fl[2] == 1 and fl[3] == 0
    # non-float64 / non-array entries: None, and _pose_arrays falls back
    odd = list(poses)
    odd[5] = RigidTransform([[1, 0, 0], [0, 1, 0], [0, 0, 1]], [1, 2, 3])
    assert _sfbhost.pack_poses(odd, R, t, fl) is None
    for got, want in zip(_pose_arrays(odd), _py_pose_arrays(odd)):
        assert np.array_equal(got, want)
    with pytest.raises(ValueError):
        _sfbhost.pack_poses(poses, R[:3], t, fl)
    # pull: fresh C-contiguous owned copies, frame 0 untouched
    ids = [10 * k for k in range(n)]
    d = {f: None for f in ids}
    assert _sfbhost.make_poses(d, ids, R, t, RigidTransform, 1) is None
    assert d[0] is None
    for k in range(1, n):
        p = d[ids[k]]
        assert type(p) is RigidTransform
        assert np.array_equal(p.rotation, R[k]) and np.array_equal(p.translation, t[k])
        assert p.rotation.flags.c_contiguous and p.rotation.flags.owndata
