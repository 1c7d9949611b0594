"""Break the end-to-end solve (public API, host inputs) into host/device phases."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_1604_01093_b200 import solver as S, synth
from paper_1604_01093_b200.runtime import runtime

sc = synth.make(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
caches = bench.pin_caches(sc.caches)
W, C = S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config)
rt = runtime(0)
for rep in range(4):
    rt.clear_frames()
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, caches); t.append(time.perf_counter())
    cl = [caches[f] for f in sc.frame_ids]
    rt.slots_for(cl); t.append(time.perf_counter())
    p._problem(); t.append(time.perf_counter())
    st = p.solve(W, C); torch.cuda.synchronize(); t.append(time.perf_counter())
    p.close(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: init {d[0]:.1f}  frames {d[1]:.1f}  problem {d[2]:.1f}  solve {d[3]:.1f}  close {d[4]:.1f} ms", flush=True)
