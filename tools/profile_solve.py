"""Run N solves of a synthetic configuration (for ncu / compute-sanitizer captures)."""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1604_01093_b200 import solver as S  # noqa: E402
from scenes import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--max-iterations", type=int, default=None)
a = ap.parse_args()
sc = synth.make(a.config)
W = S.EnergyWeights(**sc.weights)
C = S.SolverConfig(**sc.config)
p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, sc.caches)
for k in range(a.solves):
    p.poses = dict(sc.init)
    t0 = time.perf_counter()
    st = p.solve(W, C, a.max_iterations or sc.max_iterations)
    print(f"solve {k}: {1e3 * (time.perf_counter() - t0):.1f} ms wall, {len(st.iterations)} GN, "
          f"final {st.final_energy:.6e}", flush=True)
