"""Golden vectors for dense_verify, produced by the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_verify_golden.py

Scene: the cfg3 facade (synth.make("cfg3"), 100 keyframes at 80x60).  The
reference builds its own caches from the stored renders with its
build_cache (frames.py:75-151); every plane dense_verify reads (including
intensity_low) is checked bit-identical to ours, so the GPU tests can rebuild
the inputs from the deterministic synth instead of shipping them.

Pairs: neighbours at gaps 1..24 and loop closures, with transform_ij = the
truth relative pose (pose_j^-1 o pose_i) perturbed by 0 .. 0.08 rad / m, so
that both gates and the pass rule are exercised; a quarter of the rotations
are Fortran-ordered (the (m,3) @ R.T rounding order depends on the layout).
Outputs: scanfuse.filters.dense_verify (filters.py:253-277) for every pair.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from scanfuse import filters as RF  # noqa: E402
from scanfuse import frames as RFr  # noqa: E402
from scanfuse import geometry as RG  # noqa: E402

from scenes import synth  # noqa: E402


def exp_so3(w):
    th = np.linalg.norm(w)
    if th < 1e-12:
        return np.eye(3)
    k = w / th
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K


def main():
    sc = synth.make("cfg3")
    kr = RG.Intrinsics(sc.render_k.fx, sc.render_k.fy, sc.render_k.cx, sc.render_k.cy,
                       sc.render_k.width, sc.render_k.height)
    ref = {}
    for f, (g, d) in sc.renders.items():
        fr = RFr.RgbdFrame(index=f, color=np.repeat(g[..., None], 3, axis=2), depth=d)
        ref[f] = RFr.build_cache(fr, kr, sc.low_size[0], sc.low_size[1])
        ours = sc.caches[f]
        for name in ("valid_depth", "valid_normal", "points_low", "normals_low", "intensity_low"):
            a, b = np.asarray(getattr(ref[f], name)), np.asarray(getattr(ours, name))
            assert a.dtype == b.dtype and np.array_equal(a, b), (f, name)
    rng = np.random.default_rng(1604)
    ids = sc.frame_ids
    n = len(ids)
    pairs = []
    for gap in (1, 2, 3, 5, 8, 13, 24):
        for i in range(0, n - gap, 7):
            pairs.append((ids[i], ids[i + gap]))
    for i in range(0, n // 2, 9):  # out-and-back loop closures
        pairs.append((ids[i], ids[n - 1 - i]))
    out_pairs, Rs, ts, forder, noise = [], [], [], [], []
    passed, e_ij, e_ji, c_ij, c_ji = [], [], [], [], []
    cfg = RF.FilterConfig()
    for k, (a, b) in enumerate(pairs):
        Ta = RG.RigidTransform(np.array(sc.truth[a].rotation), np.array(sc.truth[a].translation))
        Tb = RG.RigidTransform(np.array(sc.truth[b].rotation), np.array(sc.truth[b].translation))
        rel = Tb.inverse() @ Ta
        s = [0.0, 0.002, 0.01, 0.03, 0.08][k % 5]
        dR = exp_so3(rng.normal(size=3) * s)
        R = dR @ rel.rotation
        t = rel.translation + rng.normal(size=3) * s
        f_order = (k % 4) == 3
        R = np.asfortranarray(R) if f_order else np.ascontiguousarray(R)
        T = RG.RigidTransform(R, t)
        r = RF.dense_verify(ref[a], ref[b], T, cfg)
        out_pairs.append((a, b))
        Rs.append(np.array(R))
        ts.append(t)
        forder.append(f_order)
        noise.append(s)
        passed.append(r.passed)
        e_ij.append(r.mean_error_ij)
        e_ji.append(r.mean_error_ji)
        c_ij.append(r.valid_count_ij)
        c_ji.append(r.valid_count_ji)
    np.savez_compressed(
        HERE / "verify.npz", pairs=np.array(out_pairs, dtype=np.int32), R=np.array(Rs),
        t=np.array(ts), f_order=np.array(forder), noise=np.array(noise),
        passed=np.array(passed), err_ij=np.array(e_ij), err_ji=np.array(e_ji),
        count_ij=np.array(c_ij, dtype=np.int64), count_ji=np.array(c_ji, dtype=np.int64))
    print(f"{len(out_pairs)} pairs, {sum(passed)} passed, counts "
          f"{min(c_ij)}..{max(c_ij)}")


if __name__ == "__main__":
    main()
