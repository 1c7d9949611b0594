"""pytest plugin: run the reference's UNMODIFIED tests against the drop-in.

Loaded with `-p shim` (tests/ref on sys.path) by
tests/test_gpu_reference_unmodified.py.  It imports the vendored reference
package (tests/ref/_vendor/scanfuse) and replaces two of its modules in
sys.modules before the test files are collected:

* `scanfuse.solver` -> every public name of `paper_1604_01093_b200.solver`
  (the B200 drop-in); anything else the tests might touch falls through to
  the reference module.
* `scanfuse.frames` -> `paper_1604_01093_b200.frames` for `build_cache`,
  `frustum_overlap`, `view_angle_deg` (device kernels), the reference's
  records (`RgbdFrame`, `CachedFrame`) and everything else.

`scanfuse.geometry` / `scanfuse.filters` stay the reference's: they only
build the tests' inputs (poses, correspondence sets).
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "_vendor"))
sys.path.insert(0, str(HERE.parent.parent))

import scanfuse  # noqa: E402  (the vendored reference package)
import scanfuse.frames as _ref_frames  # noqa: E402
import scanfuse.solver as _ref_solver  # noqa: E402

from paper_1604_01093_b200 import frames as _our_frames  # noqa: E402
from paper_1604_01093_b200 import solver as _our_solver  # noqa: E402


def _overlay(name, ours, ref, names):
    mod = types.ModuleType(name)
    mod.__doc__ = f"drop-in shim: {ours.__name__} over {ref.__name__}"
    for k in names:
        setattr(mod, k, getattr(ours, k))

    def __getattr__(attr):
        return getattr(ref, attr)

    mod.__getattr__ = __getattr__
    mod.__file__ = ours.__file__
    return mod


SOLVER_NAMES = [k for k in dir(_ref_solver) if not k.startswith("__") and hasattr(_our_solver, k)]
FRAMES_NAMES = ["build_cache", "frustum_overlap", "view_angle_deg"]

solver_shim = _overlay("scanfuse.solver", _our_solver, _ref_solver, SOLVER_NAMES)
frames_shim = _overlay("scanfuse.frames", _our_frames, _ref_frames, FRAMES_NAMES)
sys.modules["scanfuse.solver"] = solver_shim
sys.modules["scanfuse.frames"] = frames_shim
scanfuse.solver = solver_shim
scanfuse.frames = frames_shim


def pytest_report_header(config):
    missing = [k for k in dir(_ref_solver) if not k.startswith("_") and not hasattr(_our_solver, k)]
    return [f"scanfuse.solver -> {_our_solver.__file__} ({len(SOLVER_NAMES)} names; "
            f"reference-only: {', '.join(missing) or 'none'})",
            f"scanfuse.frames -> {_our_frames.__file__} ({', '.join(FRAMES_NAMES)})"]
