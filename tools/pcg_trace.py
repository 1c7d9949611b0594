"""Per-phase PCG timing on cfg4 (needs a -DPCG_TRACE build: SFB_LIB=variants/trace.so)."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_1604_01093_b200 import solver as S, _abi  # noqa: E402
from scenes import synth
sc = synth.make(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
W, Cf = S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config)
p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, sc.caches)
p.solve(W, Cf, max_iterations=1)
p.poses = dict(sc.init)
p._push_poses()
dp = p._dp
dp.build_dense_edges(60.0)
dp.linearize(W, 1.0, Cf)
for _ in range(3):
    dp.pcg(50, 0.0, 20)
buf = (C.c_ulonglong * (64 * 8))()
_abi.load().sfb_debug_pcg_trace(buf)
t = np.array(buf, dtype=np.float64).reshape(64, 8)[1:51, :5]
d = np.diff(t, axis=1) / 1e3
names = ["matvec", "reduce1", "phase2", "reduce2"]
for k, nme in enumerate(names):
    print(f"{nme:18s} {np.median(d[:, k]):7.2f} us")
it = (t[1:, 0] - t[:-1, 0]) / 1e3
print("iteration", np.median(it), "us")
