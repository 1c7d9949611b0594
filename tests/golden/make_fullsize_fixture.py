"""Full-size linearisation fixture (cfg4: 500 keyframes 160x120) from the
UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize_fixture.py

scanfuse.solver.AlignmentProblem.normal_equations (solver.py:630-660) at the
initial poses with the full dense weight (w_dense = 1, default EnergyWeights
and SolverConfig) over the reference's own dense-edge set
(tests/golden/edges_cfg4.npy).  The 15,000 edges are split over a process
pool (each worker a reference AlignmentProblem whose dense_edges is a slice;
the sparse sets ride on worker 0 only) and the additive outputs are summed:
energy, gradient, Jacobi diagonal, and A.u for a fixed random u.
"""

from __future__ import annotations

import multiprocessing as mp
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
N_WORK = 32


def _work(k):
    from scanfuse import filters as RF
    from scanfuse import geometry as RG
    from scanfuse import solver as RS
    from scenes import synth
    sc = synth.make("cfg4")
    poses = {f: RG.RigidTransform(np.array(p.rotation), np.array(p.translation))
             for f, p in sc.init.items()}
    sets = [RF.CorrespondenceSet(s.frame_i, s.frame_j, s.points_i, s.points_j,
                                 np.zeros((len(s), 2), dtype=int), None, True)
            for s in sc.corr_sets] if k == 0 else []
    edges = [tuple(int(x) for x in e) for e in np.load(HERE / "edges_cfg4.npy")]
    p = RS.AlignmentProblem(sc.frame_ids, poses, sets, sc.caches)
    p.dense_edges = edges[k::N_WORK]
    eqs, energy, _, _ = p.normal_equations(RS.EnergyWeights(), 1.0, RS.SolverConfig())
    u = np.random.default_rng(1604).normal(size=p.n_vars)
    return energy, np.asarray(eqs.gradient), np.asarray(eqs.diagonal), np.asarray(eqs.apply(u))


def main():
    t0 = time.time()
    with mp.get_context("fork").Pool() as pool:
        res = pool.map(_work, range(N_WORK))
    energy = sum(r[0] for r in res)
    grad = sum(r[1] for r in res)
    diag = sum(r[2] for r in res)
    au = sum(r[3] for r in res)
    np.savez_compressed(HERE / "fullsize_cfg4.npz", energy=energy, gradient=grad, diagonal=diag,
                        au=au, u_seed=1604)
    print(f"energy {energy:.12e}  |g| {np.linalg.norm(grad):.6e}  {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
