"""Build a tuning variant of libsfb.so into variants/NAME.so.

usage: python tools/build_variant.py NAME [--file sfb_dense.cu=PATH ...] [-- NVCC FLAGS]
Copies csrc/ to a temp dir, swaps in replacement files, compiles with the
standard flags plus the extra ones.  Select at run time with SFB_LIB=variants/NAME.so.
"""
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1604_01093_b200 import _build  # noqa: E402

name = sys.argv[1]
args = sys.argv[2:]
extra = []
if "--" in args:
    extra = args[args.index("--") + 1:]
    args = args[:args.index("--")]
repl = {}
while args:
    if args[0] == "--file":
        k, v = args[1].split("=", 1)
        repl[k] = Path(v)
        args = args[2:]
    else:
        raise SystemExit(f"bad arg {args[0]}")
out = ROOT / "variants" / f"{name}.so"
out.parent.mkdir(exist_ok=True)
with tempfile.TemporaryDirectory(dir=_build.PKG, prefix='_var_') as td:  # keeps ../../include
    td = Path(td)
    for p in _build.CSRC.iterdir():
        if p.suffix in (".cu", ".cuh"):
            shutil.copy(repl.get(p.name, p), td / p.name)
    srcs = sorted(td.glob("*.cu"))
    cmd = [_build._nvcc(), *_build.NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-o", str(out),
           *map(str, srcs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
print(out)
