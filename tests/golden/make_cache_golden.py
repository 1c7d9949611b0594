"""Golden digests of build_cache, produced by the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cache_golden.py

Inputs are regenerated deterministically by `cache_inputs()` (shared with
tests/test_gpu_cache.py): the cfg2 renders (11 frames 640x480 -> 80x60) and
adversarial frames (random colour, depth holes, NaN samples, ties, fully
invalid blocks) at block shapes 8x8, 6x6, 4x4, 2x3 and 1x1.  For every frame
the reference's scanfuse.frames.build_cache (frames.py:75-151) output planes
are hashed (sha256 of dtype, shape and bytes); the GPU test compares the
device planes against these digests.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

PLANES = ("intensity_low", "depth_low", "points_low", "normals_low", "grad_low", "valid_depth",
          "valid_normal")
K = (525.0, 525.0, 319.5, 239.5, 640, 480)


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def cache_inputs():
    """[(name, color (H,W,3) u8, depth (H,W) f32, (low_w, low_h), K)]"""
    from scenes import synth
    out = []
    sc = synth.make("cfg2")
    for f in sorted(sc.renders):
        g, d = sc.renders[f]
        out.append((f"cfg2_{f}", np.repeat(g[..., None], 3, axis=2), d, (80, 60), K))
    rng = np.random.default_rng(75151)
    for k, (W, H, lw, lh) in enumerate([(640, 480, 80, 60), (640, 480, 80, 60), (480, 360, 80, 60),
                                        (320, 240, 80, 60), (240, 120, 80, 60), (160, 120, 160, 120)]):
        col = rng.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
        yy, xx = np.mgrid[0:H, 0:W]
        dep = (1.5 + 0.002 * xx + 0.001 * yy + 0.05 * np.sin(xx / 7.0) * np.cos(yy / 5.0)
               + rng.normal(0, 0.01, (H, W))).astype(np.float32)
        dep[rng.random((H, W)) < 0.25] = 0.0               # holes
        if k % 2 == 0:
            dep[rng.random((H, W)) < 0.02] = np.nan        # NaN samples
            dep[rng.random((H, W)) < 0.02] = -1.0          # negative = invalid
        dep[: H // 6, : W // 5] = 0.0                      # fully invalid blocks
        dep[H // 2: H // 2 + H // 8] = np.round(dep[H // 2: H // 2 + H // 8], 1)  # ties
        kk = (K[0] * W / 640, K[1] * H / 480, (K[2] + 0.5) * W / 640 - 0.5,
              (K[3] + 0.5) * H / 480 - 0.5, W, H)
        out.append((f"adv{k}_{W}x{H}", col, dep, (lw, lh), kk))
    return out


def main():
    from scanfuse import frames as RFr
    from scanfuse import geometry as RG
    res = {}
    for name, col, dep, (lw, lh), kk in cache_inputs():
        k = RG.Intrinsics(*kk)
        c = RFr.build_cache(RFr.RgbdFrame(index=0, color=col, depth=dep), k, lw, lh)
        res[name] = {p: digest(getattr(c, p)) for p in PLANES}
    (HERE / "cache_digests.json").write_text(json.dumps(res, indent=1, sort_keys=True))
    print(f"{len(res)} frames")


if __name__ == "__main__":
    main()
