"""build_cache on the GPU (cache.build_cache_device, reference frames.py:75-151).

Every plane of every frame must be bit-identical to the reference's
build_cache: the device output is hashed against tests/golden/cache_digests.json
(made by the unmodified reference from the same deterministic inputs) and,
for a readable failure, diffed against this package's host build_cache.
"""

import json
import sys
from collections import defaultdict

import numpy as np
import pytest

from golden_io import GOLDEN

sys.path.insert(0, str(GOLDEN))
from make_cache_golden import PLANES, cache_inputs, digest  # noqa: E402

pytestmark = pytest.mark.gpu


def _groups():
    groups = defaultdict(list)
    for name, col, dep, low, kk in cache_inputs():
        groups[(col.shape, low, kk)].append((name, col, dep))
    return groups


def test_device_build_cache_bit_exact():
    from paper_1604_01093_b200 import cache as CA
    from paper_1604_01093_b200 import se3
    g = json.loads((GOLDEN / "cache_digests.json").read_text())
    checked = 0
    for (shape, (lw, lh), kk), items in _groups().items():
        k = se3.Intrinsics(*kk)
        frames = [CA.RgbdFrame(i, col, dep) for i, (_, col, dep) in enumerate(items)]
        dev = CA.build_cache_device(frames, k, lw, lh)
        for (name, col, dep), c in zip(items, dev):
            host = CA.build_cache(CA.RgbdFrame(0, col, dep), k, lw, lh)
            for p in PLANES:
                a, b = np.asarray(getattr(c, p)), np.asarray(getattr(host, p))
                diff = int(np.count_nonzero(~((a == b) | (np.isnan(a) & np.isnan(b)))))
                assert digest(a) == g[name][p], f"{name}.{p}: {diff} elements differ from host"
                checked += 1
            assert c.intrinsics_low == host.intrinsics_low
    assert checked == len(g) * len(PLANES)


def test_device_caches_are_resident_and_solve_like_host_caches():
    """Caches built on the device are adopted by the frame store (no upload)
    and a cfg2 solve on them reproduces the reference's golden result."""
    from golden_io import GoldenScene, pose_errors
    from paper_1604_01093_b200 import cache as CA
    from paper_1604_01093_b200 import se3, synth
    from paper_1604_01093_b200 import solver as S
    from paper_1604_01093_b200.runtime import runtime
    s = GoldenScene("cfg2")
    sc = synth.make("cfg2")
    kr = sc.render_k
    frames = [CA.RgbdFrame(f, np.repeat(sc.renders[f][0][..., None], 3, axis=2), sc.renders[f][1])
              for f in s.ids]
    dev = CA.build_cache_device(frames, se3.Intrinsics(kr.fx, kr.fy, kr.cx, kr.cy, kr.width,
                                                       kr.height), *sc.low_size)
    caches = {f: c for f, c in zip(s.ids, dev)}
    rt = runtime()
    assert all(id(c) in rt._frames for c in dev)
    p = S.AlignmentProblem(s.ids, s.init, s.corr_sets, caches)
    stats = p.solve(s.weights_obj(S), s.config_obj(S), s.max_iterations)
    ref = {f: se3.RigidTransform(s.g["final_R"][k], s.g["final_t"][k]) for k, f in enumerate(s.ids)}
    re, te = pose_errors(p.poses, ref)
    assert re < 1e-4 and te < 1e-4
    e_ref = s.g["records"][-1][1]
    assert abs(stats.final_energy - e_ref) <= 1e-5 * abs(e_ref)


def test_dense_verify_on_device_caches_matches_host_caches():
    from paper_1604_01093_b200 import cache as CA
    from paper_1604_01093_b200 import filters as F
    from paper_1604_01093_b200 import se3, synth
    sc = synth.make("cfg2")
    kr = sc.render_k
    k = se3.Intrinsics(kr.fx, kr.fy, kr.cx, kr.cy, kr.width, kr.height)
    ids = sorted(sc.renders)
    frames = [CA.RgbdFrame(f, np.repeat(sc.renders[f][0][..., None], 3, axis=2), sc.renders[f][1])
              for f in ids]
    dev = dict(zip(ids, CA.build_cache_device(frames, k, *sc.low_size)))
    pairs = [(a, b) for a in ids for b in ids if a < b]
    T = {p: sc.truth[p[1]].inverse().compose(sc.truth[p[0]]) for p in pairs}
    r_dev = F.dense_verify_many([(dev[a], dev[b], T[(a, b)]) for a, b in pairs], F.FilterConfig())
    r_host = F.dense_verify_many([(sc.caches[a], sc.caches[b], T[(a, b)]) for a, b in pairs],
                                 F.FilterConfig())
    assert r_dev == r_host
