"""Copy recipe: the reference's own solver-path tests (and the reference
package they import) into tests/ref/_vendor/, UNMODIFIED.

    python tests/ref/vendor.py            # in the build container (needs /root/reference)

Test infrastructure only.  `_vendor/` is git-ignored (no reference source
enters the history) but not gpurun-ignored, so the copies travel to the GPU
box with the built libraries; `__graft_entry__.build()` refreshes them
whenever /root/reference is present.  tests/test_gpu_reference_unmodified.py
runs them there through the import shim in tests/ref/shim.py.
"""

from __future__ import annotations

import hashlib
import json
import shutil
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent / "_vendor"
TESTS = ("test_solver.py", "test_frames.py")


def vendor(ref: Path = REF, out: Path = OUT) -> bool:
    if not (ref / "src" / "scanfuse" / "solver.py").exists():
        return False
    if out.exists():
        shutil.rmtree(out)
    (out / "scanfuse").mkdir(parents=True)
    manifest = {}
    for src in sorted((ref / "src" / "scanfuse").glob("*.py")):
        shutil.copy2(src, out / "scanfuse" / src.name)
        manifest[f"scanfuse/{src.name}"] = hashlib.sha256(src.read_bytes()).hexdigest()
    for name in TESTS:
        shutil.copy2(ref / "tests" / name, out / name)
        manifest[name] = hashlib.sha256((ref / "tests" / name).read_bytes()).hexdigest()
    (out / "MANIFEST.json").write_text(json.dumps(manifest, indent=1) + "\n")
    return True


if __name__ == "__main__":
    ok = vendor()
    print("vendored" if ok else "reference not present", OUT)
    sys.exit(0 if ok else 1)
