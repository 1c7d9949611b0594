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
    from paper_1604_01093_b200 import synth
    a, b = synth.make("cfg2"), synth.make("cfg2")
    assert synth.cache_digest(a.caches) == synth.cache_digest(b.caches)
    assert all(np.array_equal(x.points_i, y.points_i) for x, y in zip(a.corr_sets, b.corr_sets))


def test_build_cache_matches_reference_fixture():
    from golden_io import GoldenScene
    s = GoldenScene("cfg2")
    assert s.cache_sha_ok
