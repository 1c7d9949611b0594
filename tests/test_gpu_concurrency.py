"""Concurrent use of one device context (reference contracts: "distinct
problems may be solved concurrently", solver.py:551-552; pair filtering and
dense verification are pair-parallel) and the frame store's lifetime.

* N threads calling dense_verify_many at once each get their serial result.
* Two AlignmentProblem.solve calls on different scenes at once (each stacks
  its correspondence sets through the runtime's shared pinned staging) give
  their serial results bit for bit.
* Caches the caller drops are released from the device frame store once no
  live problem uses them; clear_frames() defers slots a live problem holds.
"""

import gc
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_threads(fns):
    out = [None] * len(fns)
    err = []

    def wrap(k, fn):
        try:
            out[k] = fn()
        except BaseException as e:  # re-raised below
            err.append(e)

    ths = [threading.Thread(target=wrap, args=(k, fn)) for k, fn in enumerate(fns)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]
    return out


def test_concurrent_dense_verify_matches_serial():
    from paper_1604_01093_b200 import filters as F
    from scenes import synth
    sc = synth.make("cfg3")
    rng = np.random.default_rng(3)
    batches = []
    for b in range(6):
        pairs = []
        for _ in range(40):
            i, j = sorted(rng.choice(len(sc.frame_ids), 2, replace=False))
            fi, fj = sc.frame_ids[i], sc.frame_ids[j]
            T = sc.truth[fj].inverse().compose(sc.truth[fi])
            pairs.append((sc.caches[fi], sc.caches[fj], T))
        batches.append(pairs)
    cfg = F.FilterConfig()
    serial = [F.dense_verify_many(p, cfg) for p in batches]
    for _ in range(3):
        par = _run_threads([lambda p=p: F.dense_verify_many(p, cfg) for p in batches])
        assert par == serial


def _solve(sc):
    from paper_1604_01093_b200 import solver as S
    p = S.AlignmentProblem(sc.frame_ids, sc.init, sc.corr_sets, sc.caches)
    st = p.solve(S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config), sc.max_iterations)
    R = np.stack([np.asarray(p.poses[f].rotation) for f in sc.frame_ids])
    t = np.stack([np.asarray(p.poses[f].translation) for f in sc.frame_ids])
    p.close()
    return R, t, [(r.energy_before, r.energy_after, r.pcg_iterations) for r in st.iterations]


def test_concurrent_solves_match_serial():
    from scenes import synth
    a, b = synth.make("cfg3"), synth.make("cfg2")
    sa, sb = _solve(a), _solve(b)
    for _ in range(2):
        pa, pb = _run_threads([lambda: _solve(a), lambda: _solve(b)])
        for got, want in ((pa, sa), (pb, sb)):
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
            assert got[2] == want[2]


def test_frame_store_releases_dropped_caches():
    from paper_1604_01093_b200 import solver as S
    from scenes import synth
    from paper_1604_01093_b200.runtime import runtime
    rt = runtime(0)
    rt.clear_frames()
    base = rt.resident_frames()
    sc = synth.make("cfg2")
    ids = sc.frame_ids

    def fresh():  # new cache objects with the same planes (new identities)
        return {f: synth.CachedFrame(c.index, c.intensity_low, c.grad_low.copy(), c.depth_low,
                                     c.points_low.copy(), c.normals_low.copy(), c.intrinsics_low,
                                     c.valid_depth.copy(), c.valid_normal.copy())
                for f, c in sc.caches.items()}

    # a session over many batches of frames: dropped batches are released
    for _ in range(5):
        caches = fresh()
        S.build_dense_edges(ids, sc.init, caches, S.SolverConfig())
        assert rt.resident_frames() == base + len(ids)
        del caches
        gc.collect()
        assert rt.resident_frames() == base
    # a live problem keeps its slots through clear_frames(); they go when it closes
    caches = fresh()
    p = S.AlignmentProblem(ids, sc.init, sc.corr_sets, caches)
    st1 = p.solve(S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config), 2)
    rt.clear_frames()
    assert rt.resident_frames() == base + len(ids)
    st2 = p.solve(S.EnergyWeights(**sc.weights), S.SolverConfig(**sc.config), 2)
    assert len(st2.iterations) == len(st1.iterations)
    p.close()
    assert rt.resident_frames() == base
    # the same objects upload again after clear_frames()
    S.build_dense_edges(ids, sc.init, caches, S.SolverConfig())
    assert rt.resident_frames() == base + len(ids)
    del caches, p
    gc.collect()
    assert rt.resident_frames() == base
