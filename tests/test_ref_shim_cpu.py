"""CPU check of the reference-suite shim (tests/ref/shim.py): the vendored,
unmodified reference test files collect with `scanfuse.solver` /
`scanfuse.frames` resolving to the drop-in (no kernels run here)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parent / "ref"
VENDOR = REF / "_vendor"


def test_shim_collects_reference_suite():
    if not (VENDOR / "test_solver.py").exists():
        pytest.skip("tests/ref/_vendor missing")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), env.get("PYTHONPATH", "")])
    probe = ("import shim, scanfuse.solver as s, scanfuse.frames as f; "
             "import paper_1604_01093_b200.solver as o, paper_1604_01093_b200.frames as of; "
             "assert s.AlignmentProblem is o.AlignmentProblem and s.pcg_solve is o.pcg_solve; "
             "assert f.frustum_overlap is of.frustum_overlap and f.build_cache is of.build_cache; "
             "print('ok')")
    res = subprocess.run([sys.executable, "-c", probe], cwd=VENDOR, env=env, capture_output=True,
                         text=True, timeout=300)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]
    res = subprocess.run([sys.executable, "-m", "pytest", "-p", "shim", "-q", "-p", "no:cacheprovider",
                          "--rootdir", str(VENDOR), "--confcutdir", str(VENDOR), "--collect-only",
                          "test_solver.py", "test_frames.py"],
                         cwd=VENDOR, env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "39 tests collected" in res.stdout
