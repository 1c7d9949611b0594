"""build_cache throughput: device batch (cache.build_cache_device) vs host NumPy.

    python tools/bench_cache.py [--frames 500] [--reps 5]

Synthetic 640x480 RGB-D frames (random colour, smooth depth with holes) ->
80x60 caches.  Prints one JSON line: frames/s through the public device API
(host frames in, host CachedFrames out, planes left resident in the frame
store), the bytes it moves, and the host NumPy build_cache frames/s (1 core).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1604_01093_b200 import cache as CA, se3  # noqa: E402
from paper_1604_01093_b200.runtime import runtime  # noqa: E402
from scenes import host_cache  # noqa: E402  (the NumPy restatement, timed beside the device path)

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=500)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
rng = np.random.default_rng(0)
H, W = 480, 640
K = se3.Intrinsics(525.0, 525.0, 319.5, 239.5, W, H)
yy, xx = np.mgrid[0:H, 0:W]
frames = []
for i in range(a.frames):
    col = rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
    dep = (1.5 + 0.002 * xx + 0.001 * yy + 0.1 * np.sin((xx + i) / 9.0)).astype(np.float32)
    dep[rng.random((H, W)) < 0.1] = 0.0
    frames.append(CA.RgbdFrame(i, col, dep))
rt = runtime()
CA.build_cache_device(frames[:8], K)
ts = []
for _ in range(a.reps):
    rt.clear_frames()
    t0 = time.perf_counter()
    CA.build_cache_device(frames, K)
    ts.append(time.perf_counter() - t0)
dt = float(np.median(ts))
t0 = time.perf_counter()
ns = 8
for f in frames[:ns]:
    host_cache.build_cache(f, K)
host = (time.perf_counter() - t0) / ns
print(json.dumps({"metric": "build_cache frames/s (640x480 -> 80x60)", "frames": a.frames,
                  "device_api_ms": 1e3 * dt, "device_frames_per_s": a.frames / dt,
                  "h2d_bytes": a.frames * H * W * 7, "d2h_bytes": a.frames * 80 * 60 * 42,
                  "host_numpy_frames_per_s": 1.0 / host, "host_cores": 1}))
