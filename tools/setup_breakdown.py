"""Time the pieces of AlignmentProblem._problem (frames upload thread, set
stacking, sfb_problem_create) and the constructor, per config."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1604_01093_b200 import device_problem as DPm, solver as S  # noqa: E402
from scenes import synth
from paper_1604_01093_b200.runtime import runtime  # noqa: E402

sc = synth.make(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
caches = bench.pin_caches(sc.caches)
rt = runtime(0)
T = {}


def timed(name, fn):
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            T[name] = T.get(name, 0.0) + (time.perf_counter() - t) * 1e3
    return w


S._set_layout = timed("set_layout", S._set_layout)
rt.slots_for = timed("slots_for(upload)", rt.slots_for)
orig_create = DPm.DeviceProblem.__init__
DPm.DeviceProblem.__init__ = timed("DeviceProblem.__init__", orig_create)
for rep in range(4):
    rt.clear_frames()
    torch.cuda.synchronize()
    T.clear()
    t0 = time.perf_counter()
    p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, caches)
    t1 = time.perf_counter()
    p._problem()
    t2 = time.perf_counter()
    p.close()
    print(f"rep {rep}: ctor {(t1 - t0) * 1e3:.1f} ms, _problem {(t2 - t1) * 1e3:.1f} ms;",
          {k: round(v, 2) for k, v in T.items()}, flush=True)
