"""Dense-edge list of a synthetic config from the device pair filter -> gpurun_out/edges_<cfg>.npy."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
from paper_1604_01093_b200 import solver as S  # noqa: E402
from scenes import synth
for name in sys.argv[1:]:
    sc = synth.make(name)
    e = np.array(S.build_dense_edges(sc.frame_ids, sc.init, sc.caches, S.SolverConfig()), dtype=np.int32)
    Path("gpurun_out").mkdir(exist_ok=True)
    np.save(f"gpurun_out/edges_{name}.npy", e)
    print(name, len(e))
