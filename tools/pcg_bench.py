"""Time the device PCG alone on a linearised configuration (per-iteration cost)."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1604_01093_b200 import solver as S
from scenes import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
a = ap.parse_args()
sc = synth.make(a.config)
W, C = S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config)
p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, sc.caches)
p.solve(W, C, max_iterations=1)
p.poses = dict(sc.init)
p._push_poses()
pairs = p._dp.build_dense_edges(60.0)
dp = p._dp
dp.linearize(W, 1.0, C)
for it in (1, 2, 5, 10, 20, 50):
    dp.pcg(it, 0.0, 20)
    t0 = time.perf_counter()
    n = 20
    for _ in range(n):
        res = dp.pcg(it, 0.0, 20)
    dt = (time.perf_counter() - t0) / n
    print(f"max_it {it:3d}: {dt*1e6:8.1f} us/call  iters={res[0]}  rel={res[1]:.3e}", flush=True)
