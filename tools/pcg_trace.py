import ctypes as C, os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_1604_01093_b200 import solver as S, synth, _abi
sc = synth.make("cfg4")
W, Cf = S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config)
p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, sc.caches)
p.solve(W, Cf, max_iterations=1)
p.poses = dict(sc.init); p._push_poses()
dp = p._dp
dp.build_dense_edges(60.0)
dp.linearize(W, 1.0, Cf)
for _ in range(3): dp.pcg(50, 0.0, 20)
buf = (C.c_ulonglong * (64 * 8))()
_abi.load().sfb_debug_pcg_trace(buf)
t = np.array(buf, dtype=np.float64).reshape(64, 8)[1:51]
d = np.diff(t, axis=1) / 1e3
names = ["matvec", "blk_sum", "barrier1", "allsum+alpha", "phase2", "barrier2", "allsum2"]
for k, nme in enumerate(names): print(f"{nme:14s} {np.median(d[:, k]):7.2f} us")
it = (t[1:, 0] - t[:-1, 0]) / 1e3
print("iteration", np.median(it), "us")
