"""Break the end-to-end solve (public API, host inputs) into host/device phases."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1604_01093_b200 import solver as S  # noqa: E402
from scenes import synth
from paper_1604_01093_b200.device_problem import DeviceProblem  # noqa: E402
from paper_1604_01093_b200.runtime import runtime  # noqa: E402

sc = synth.make(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
caches = bench.pin_caches(sc.caches)
W, C = S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config)
rt = runtime(0)
for rep in range(4):
    rt.clear_frames()
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, caches); t.append(time.perf_counter())
    p._problem(); t.append(time.perf_counter())  # frame upload || set stacking, problem create
    st = p.solve(W, C); torch.cuda.synchronize(); t.append(time.perf_counter())
    p.close(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: init {d[0]:.1f}  frames+problem {d[1]:.1f}  solve {d[2]:.1f}  close {d[3]:.1f}"
          f"  total {sum(d):.1f} ms", flush=True)

# raw host->device copy rates for reference
n = 341 * 1024 * 1024
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"pinned H2D 341 MiB: {dt*1e3:.2f} ms = {n/dt/1e9:.1f} GB/s")
pg = torch.empty(n // 4, dtype=torch.uint8)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dst[: n // 4].copy_(pg); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"pageable H2D 85 MiB: {dt*1e3:.2f} ms = {n/4/dt/1e9:.1f} GB/s")
