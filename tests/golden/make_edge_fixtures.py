"""Full-size dense-edge fixtures (cfg4: 500 keyframes 160x120, cfg5: 2000 at
80x60) from the UNMODIFIED reference's pair filter.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_edge_fixtures.py cfg4 cfg5

The reference's build_dense_edges (solver.py:130-148) visits every pair
a < b with view_angle_deg / frustum_overlap (frames.py:154-188); that is
~2.5 CPU-minutes at cfg4 and ~7 at cfg5, so the same per-pair predicate of the
reference is evaluated here on a process pool and the accepted pairs are
emitted in build_dense_edges' order.  Inputs: synth.make(cfg) (deterministic)
at its initial poses, default SolverConfig (60 degrees).
"""

from __future__ import annotations

import multiprocessing as mp
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

_S = {}


def _scene(name):
    if name not in _S:
        from scenes import synth
        from scanfuse import geometry as RG
        sc = synth.make(name)
        poses = {f: RG.RigidTransform(np.array(p.rotation), np.array(p.translation))
                 for f, p in sc.init.items()}
        _S[name] = (sc, poses)
    return _S[name]


def _work(args):
    from scanfuse import frames as RFr
    name, chunk, max_deg = args
    sc, poses = _scene(name)
    ids = sc.frame_ids
    out = []
    for a, b in chunk:
        i, j = ids[a], ids[b]
        if RFr.view_angle_deg(poses[i], poses[j]) >= max_deg:
            continue
        if RFr.frustum_overlap(sc.caches[i], poses[i], sc.caches[j], poses[j]) <= 0.0:
            continue
        if RFr.frustum_overlap(sc.caches[j], poses[j], sc.caches[i], poses[i]) <= 0.0:
            continue
        out.append((a, b))
    return out


def main(names):
    from scanfuse import solver as RS
    max_deg = RS.SolverConfig().view_angle_max_deg
    for name in names:
        sc, _ = _scene(name)
        n = len(sc.frame_ids)
        pairs = [(a, b) for a in range(n) for b in range(a + 1, n)]
        chunks = [(name, pairs[k::64], max_deg) for k in range(64)]
        with mp.get_context("fork").Pool() as pool:
            res = pool.map(_work, chunks)
        acc = sorted(e for r in res for e in r)  # build_dense_edges' (a, b) loop order
        ids = sc.frame_ids
        edges = np.array([(ids[a], ids[b]) for a, b in acc], dtype=np.int32).reshape(-1, 2)
        np.save(HERE / f"edges_{name}.npy", edges)
        print(name, len(edges))


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg4", "cfg5"])
