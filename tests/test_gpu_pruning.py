"""solve_with_pruning with the device problem resident across prune rounds
(sfb_problem_drop_sets + per-set maxima of the live problem) against the
reference's round structure (solver.py:779-816): a fresh AlignmentProblem per
round over the surviving sets and max_residual_set (:765-776) on a separate
sparse problem.  Both must agree bit-for-bit."""

import numpy as np
import pytest

from paper_1604_01093_b200 import solver as S
from scenes import synth
from paper_1604_01093_b200.se3 import RigidTransform
from scenes.synth import chunk_corr_sets, chunk_ground_truth, make_corr_set

pytestmark = pytest.mark.gpu


def fresh_rounds(frame_ids, poses, corr_sets, weights, config, caches=None):
    """The reference's loop: a new problem per round, max_residual_set after it."""
    sets = list(corr_sets)
    poses = dict(poses)
    removed, invalid, stats = [], [], []
    rounds, r_max = 0, 0.0
    while True:
        rounds += 1
        connected = {f for cs in sets for f in (cs.frame_i, cs.frame_j)}
        active = [f for f in frame_ids if f in connected]
        invalid.extend(f for f in frame_ids if f not in connected and f not in invalid)
        if len(active) < 2 or not sets:
            r_max = 0.0
            break
        prob = S.AlignmentProblem(active, poses, sets, caches)
        stats.append(prob.solve(weights, config))
        poses.update(prob.poses)
        prob.close()
        worst, r_max = S.max_residual_set(poses, sets)
        if r_max <= config.prune_residual_max:
            break
        off = sets.pop(worst)
        removed.append((off.frame_i, off.frame_j))
    return poses, sets, S.PruneReport(removed, invalid, rounds, r_max), stats


def _records(stats):
    return [[(r.energy_before, r.energy_after, r.pcg_iterations, r.pcg_residual, r.accepted)
             for r in st.iterations] for st in stats]


def _check(ids, a, b):
    pa, ka, ra, sa = a
    pb, kb, rb, sb = b
    assert ra == rb
    assert [(c.frame_i, c.frame_j) for c in ka] == [(c.frame_i, c.frame_j) for c in kb]
    assert _records(sa) == _records(sb)
    for f in ids:
        assert np.array_equal(np.asarray(pa[f].rotation), np.asarray(pb[f].rotation))
        assert np.array_equal(np.asarray(pa[f].translation), np.asarray(pb[f].translation))


def test_resident_pruning_matches_fresh_rounds_sparse():
    rng = np.random.default_rng(31)
    truth, world = chunk_ground_truth(rng, n_frames=7)
    sets = chunk_corr_sets(rng, truth, world, per_pair=15, noise=0.001)
    bad = []
    for (i, j, shift) in ((1, 4, 0.5), (2, 6, 0.3), (0, 5, 0.2)):
        p = rng.uniform(-0.5, 0.5, size=(8, 3)) + np.array([0, 0, 2.0])
        bad.append(make_corr_set(i, j, p, p + np.array([shift, 0.0, 0.0])))
    all_sets = sets[:5] + [bad[0]] + sets[5:12] + [bad[1]] + sets[12:] + [bad[2]]
    init = {i: RigidTransform.identity() for i in range(7)}
    W = S.EnergyWeights(sparse=1.0, photo=0.0, geo=0.0)
    C = S.SolverConfig()
    a = S.solve_with_pruning(list(range(7)), init, all_sets, W, C)
    b = fresh_rounds(list(range(7)), init, all_sets, W, C)
    assert len(a[2].removed_pairs) >= 2, a[2]
    _check(range(7), a, b)


def test_resident_pruning_orphaned_frame_rebuilds():
    # pruning the only set of frame 2 disconnects it: the next round is a new
    # problem over the remaining frames, exactly as in the reference
    rng = np.random.default_rng(32)
    p = rng.uniform(-0.5, 0.5, size=(10, 3)) + np.array([0, 0, 2.0])
    sets = [make_corr_set(0, 1, p, p), make_corr_set(1, 3, p, p + 0.001),
            make_corr_set(1, 2, p, p + np.array([0.4, 0.0, 0.0]))]
    init = {i: RigidTransform.identity() for i in range(4)}
    W = S.EnergyWeights(sparse=1.0, photo=0.0, geo=0.0)
    C = S.SolverConfig()
    a = S.solve_with_pruning([0, 1, 2, 3], init, sets, W, C)
    b = fresh_rounds([0, 1, 2, 3], init, sets, W, C)
    _check(range(4), a, b)


def test_resident_pruning_with_dense_terms():
    sc = synth.make("cfg2")
    ids = sc.frame_ids
    rng = np.random.default_rng(33)
    p = rng.uniform(-0.5, 0.5, size=(8, 3)) + np.array([0, 0, 2.0])
    bad = make_corr_set(ids[2], ids[7], p, p + np.array([0.6, 0.0, 0.0]))
    sets = list(sc.corr_sets) + [bad]
    W = S.EnergyWeights(**sc.weights)
    C = S.SolverConfig(**sc.config)
    a = S.solve_with_pruning(ids, sc.init, sets, W, C, caches=sc.caches)
    b = fresh_rounds(ids, sc.init, sets, W, C, caches=sc.caches)
    assert (ids[2], ids[7]) in a[2].removed_pairs
    _check(ids, a, b)
