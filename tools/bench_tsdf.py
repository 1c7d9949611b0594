"""TSDF integrate / de-integrate throughput on the GPU vs the CPU oracle.

    python tools/bench_tsdf.py [--voxel 0.004] [--frames 11] [--reps 3]

The cfg2 RGB-D sequence (640x480, ground-truth poses) integrated into one
volume and de-integrated again through the public API (host frames in).
Prints one JSON line: ms per integrate and per de-integrate, touched blocks
and voxel updates per second, and the NumPy oracle's seconds per integrate on
one core (first frame only: it takes seconds).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
from make_tsdf_golden import tsdf_inputs  # noqa: E402

from paper_1604_01093_b200 import se3  # noqa: E402
from paper_1604_01093_b200 import tsdf as T  # noqa: E402
from paper_1604_01093_b200.cache import RgbdFrame  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--voxel", type=float, default=0.004)
ap.add_argument("--frames", type=int, default=11)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-cpu", action="store_true")
a = ap.parse_args()
frames, K, truth, _ = tsdf_inputs()
k = se3.Intrinsics(*K)
fr = [RgbdFrame(i, c, d) for i, (c, d) in enumerate(frames[:a.frames])]
poses = [se3.RigidTransform(*truth[i]) for i in range(len(fr))]
v = T.TsdfVolume(a.voxel)
v.integrate(fr[0], k, poses[0])
v.deintegrate(fr[0], k, poses[0])
ti, td = [], []
for _ in range(a.reps):
    for f, p in zip(fr, poses):
        t0 = time.perf_counter()
        v.integrate(f, k, p)
        ti.append(time.perf_counter() - t0)
    nb = len(v)
    for f, p in zip(fr, poses):
        t0 = time.perf_counter()
        v.deintegrate(f, k, p)
        td.append(time.perf_counter() - t0)
    assert len(v) == 0
cpu = None
if not a.no_cpu:
    from oracle import scanfuse_oracle as O
    o = O.TsdfOracle(a.voxel)
    t0 = time.perf_counter()
    o.apply_frame(frames[0][0], frames[0][1], k, truth[0], 1)
    cpu = time.perf_counter() - t0
print(json.dumps({"metric": "TSDF integrate ms per 640x480 frame", "voxel_size": a.voxel,
                  "frames": len(fr), "integrate_ms": 1e3 * float(np.median(ti)),
                  "deintegrate_ms": 1e3 * float(np.median(td)), "blocks_after_all": nb,
                  "cpu_oracle_integrate_s": cpu, "cpu_cores": 1}))
