"""Throughput of dense_verify (filters.py:216-277) on the GPU vs the CPU oracle.

    python tools/bench_verify.py [--config cfg4] [--pairs N] [--reps 5]

Workload: the config's scene, every dense edge (frame pair that passes the
solver's overlap filter) checked with its ground-truth relative transform,
i.e. the two-sided verification of all candidate loop closures at once.
Prints one JSON line: pairs/s through the public API (`dense_verify_many`,
host transforms in, results out) and through the bare C call, the kernel's
source-plane bytes per direction, and the oracle's single-core pairs/s on a
sample.
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1604_01093_b200 import _abi  # noqa: E402
from scenes import synth
from paper_1604_01093_b200 import filters as F  # noqa: E402
from paper_1604_01093_b200 import solver as S  # noqa: E402
from paper_1604_01093_b200.runtime import runtime  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--pairs", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--cpu-sample", type=int, default=40)
a = ap.parse_args()

sc = synth.make(a.config)
edges = list(S.build_dense_edges(sc.frame_ids, sc.truth, sc.caches, S.SolverConfig()))
if a.pairs:
    edges = edges[:a.pairs]
pairs = [(sc.caches[i], sc.caches[j], sc.truth[j].inverse().compose(sc.truth[i])) for i, j in edges]
cfg = F.FilterConfig()
res = F.dense_verify_many(pairs, cfg)  # warm-up: uploads planes + intensity

t_api = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    res = F.dense_verify_many(pairs, cfg)
    t_api.append(time.perf_counter() - t0)

# bare C call (same inputs), synchronous: H2D of items + kernel + D2H
rt = runtime()
slots = rt.intensity_slots_for([c for p in pairs for c in p[:2]])
n = 2 * len(pairs)
src = np.array([slots[2 * (k // 2) + (k % 2)] for k in range(n)], dtype=np.int32)
dst = np.array([slots[2 * (k // 2) + 1 - (k % 2)] for k in range(n)], dtype=np.int32)
R9 = np.repeat(np.stack([np.asarray(T.rotation).reshape(9) for _, _, T in pairs]), 2, axis=0)
t3 = np.repeat(np.stack([np.asarray(T.translation) for _, _, T in pairs]), 2, axis=0)
flags = np.zeros(n, dtype=np.uint8)
flags[1::2] = 1
from paper_1604_01093_b200._rounding import probe  # noqa: E402
pr = probe()
vc = _abi.VerifyConfig(cfg.verify_depth_max, cfg.verify_normal_min, cfg.verify_color_max,
                       pr["apply_n"], pr["apply_1"], pr["apply_nf"], pr["apply_1f"])
err = np.zeros(n)
cnt = np.zeros(n, dtype=np.int64)
t_c = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    _abi.check(rt.lib.sfb_dense_verify(rt.handle, n, _abi.ptr(src), _abi.ptr(dst), _abi.ptr(R9),
                                       _abi.ptr(t3), _abi.ptr(flags),
                                       _abi.C.byref(vc), _abi.ptr(err), _abi.ptr(cnt)), rt.handle)
    t_c.append(time.perf_counter() - t0)

# CPU oracle sample (single core)
from oracle import scanfuse_oracle as O  # noqa: E402
sample = pairs[:: max(1, len(pairs) // a.cpu_sample)][:a.cpu_sample]
t0 = time.perf_counter()
for ci, cj, T in sample:
    O.dense_verify(ci, cj, (np.asarray(T.rotation), np.asarray(T.translation)))
cpu_s = (time.perf_counter() - t0) / len(sample)

hw = sc.low_size[0] * sc.low_size[1]
# per direction: the source pixel plane read once (P 16 B) + N and I of the
# eligible pixels (20 B) + the gathered target P, N (32 B) and 4 intensity taps
# (16 B) of each associated pixel: upper bound 84 B/px
line = {
    "metric": "dense_verify pairs/s (two-sided)", "config": a.config, "pairs": len(pairs),
    "resolution": list(sc.low_size), "passed": int(sum(r.passed for r in res)),
    "api_pairs_per_s": len(pairs) / float(np.median(t_api)),
    "api_ms": 1e3 * float(np.median(t_api)),
    "c_call_ms": 1e3 * float(np.median(t_c)),
    "c_pairs_per_s": len(pairs) / float(np.median(t_c)),
    "bytes_per_direction_upper": 84 * hw,
    "c_call_gbs_upper": 2 * len(pairs) * 84 * hw / float(np.median(t_c)) / 1e9,
    "cpu_oracle_pairs_per_s": 1.0 / cpu_s, "cpu_cores": 1, "cpu_sample": len(sample),
    "launches": _abi.launch_count(),
}
print(json.dumps(line))
