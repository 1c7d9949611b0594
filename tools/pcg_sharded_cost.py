"""Per-iteration cost of the sharded-PCG machinery on ONE GPU: the partial
matvec + single-block scalar update (sfb_pcg_sharded) with a one-rank NCCL
all-reduce, against the persistent replicated PCG kernel on the same system.
The one-rank all-reduce is a local no-op copy, so this isolates the device
side; the NVLink collective latency adds to it on a real multi-GPU box."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_1604_01093_b200 import solver as S  # noqa: E402
from scenes import synth
from paper_1604_01093_b200.shard import ShardComm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
sc = synth.make(cfg)
W, C = S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config)
p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, sc.caches)
p.solve(W, C, max_iterations=1)
dp = p._dp
comm = ShardComm(pcg="sharded")
dp.build_dense_edges(C.view_angle_max_deg)
dp.linearize(W, 1.0, C)
ar = comm.pcg_allreduce(dp)
calls = [0]


def counted(ptr, n, stream):
    calls[0] += 1
    ar(ptr, n, stream)


out = {}
for name, fn in (("replicated (persistent kernel)", lambda: dp.pcg(50, 0.0, 20)),
                 ("sharded (matvec + NCCL + update)", lambda: dp.pcg_sharded(50, 0.0, 20, counted))):
    fn()
    torch.cuda.synchronize()
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    out[name] = (time.perf_counter() - t0) / reps * 1e3 / 50 * 1e3
    print(f"{cfg} {name}: {out[name]:.1f} us per iteration (wall), result {r}", flush=True)
print(f"all-reduce calls per sharded PCG: {calls[0] // (reps + 1)}")
dist.destroy_process_group()
