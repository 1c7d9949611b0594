"""Pixel accounting of one fused dense pass (needs a -DDENSE_COUNT build:
SFB_LIB=variants/count.so): how many source pixels are processed vs associated."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1604_01093_b200 import _abi, solver as S  # noqa: E402
from scenes import synth
sc = synth.make(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
W, Cf = S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config)
p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, sc.caches)
p.solve(W, Cf, max_iterations=1)
dp = p._dp
buf = (C.c_ulonglong * 8)()
_abi.load().sfb_debug_dense_count(buf, 1)
dp.linearize(W, 1.0, Cf)
_abi.load().sfb_debug_dense_count(buf, 1)
names = ["live&visible-tile px", "photo candidates", "photo associated", "geo candidates",
         "geo associated", "live px of active tiles", "thread slots of active tiles"]
for k, nme in enumerate(names):
    print(f"{nme:30s} {buf[k]:14d}")
print(f"directed edges {len(p.dense_edges)}  px/edge all {19200}")
