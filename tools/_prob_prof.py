import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_1604_01093_b200 import solver as S, synth
from paper_1604_01093_b200.device_problem import DeviceProblem
from paper_1604_01093_b200.runtime import runtime
name = sys.argv[1]
sc = synth.make(name)
caches = bench.pin_caches(sc.caches)
rt = runtime(0)
cl = [caches[f] for f in sc.frame_ids]
index = {f: k for k, f in enumerate(sc.frame_ids)}
for rep in range(3):
    rt.clear_frames(); torch.cuda.synchronize()
    t0 = time.perf_counter(); rt.slots_for(cl); t1 = time.perf_counter()
    lay = S._set_layout(sc.corr_sets, index, rt); t2 = time.perf_counter()
    frames, off, pi, pj = lay
    dp = DeviceProblem(len(sc.frame_ids), cl, frames, pi, pj, off); t3 = time.perf_counter()
    dp.close()
    print(f"{name} rep {rep}: upload {1e3*(t1-t0):.1f}  layout {1e3*(t2-t1):.1f}  create {1e3*(t3-t2):.1f} ms  sets {len(sc.corr_sets)}")
