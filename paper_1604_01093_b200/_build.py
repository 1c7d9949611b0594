"""Build libsfb.so in-tree with nvcc for sm_100a (no GPU needed to compile)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libsfb.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


HOST_SRC = CSRC / "host" / "sfbhost.c"


def host_module_path() -> Path:
    import sysconfig
    return PKG / ("_sfbhost" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_host(force: bool = False) -> Path:
    """The CPython helper module (_sfbhost: correspondence-set stacking) with gcc."""
    import sysconfig
    out = host_module_path()
    if not force and out.exists() and out.stat().st_mtime >= HOST_SRC.stat().st_mtime:
        return out
    tmp = out.with_suffix(".tmp")
    import numpy
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-Wall",
           "-I", sysconfig.get_paths()["include"], "-I", numpy.get_include(), str(HOST_SRC),
           "-o", str(tmp), "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, out)
    return out


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def needs_rebuild() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "sfb.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          extra: list[str] | None = None) -> Path:
    """Compile libsfb.so (or a tuning variant at `out` with `extra` nvcc flags)."""
    lib = Path(out) if out else LIB
    if out is None:
        build_host(force)
    if out is None and not force and not needs_rebuild():
        return LIB
    tmp = lib.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, *(extra or []), "-I", str(ROOT / "include"), "-o", str(tmp),
           *map(str, sources())]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
