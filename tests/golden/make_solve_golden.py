"""Full-solve goldens at the benchmarked sizes (cfg4: 500 keyframes 160x120,
cfg5: 2000 keyframes 80x60), and stride / bidirectional variants of cfg2 /
cfg3, from the UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_solve_golden.py cfg4 [cfg5 cfg2s cfg3b ...]

Test infrastructure only (never imported by the product package).

The reference's own ``AlignmentProblem.solve`` (solver.py:681-750) runs
unmodified in this process.  Only the per-directed-edge work of
``_dense_blocks`` (solver.py:582-613) and of the dense part of
``_energy_with_frozen_associations`` (:662-672) is farmed out to persistent
worker processes, each of which calls the reference's own
``associate_photo`` / ``associate_geo`` / ``photo_linearize`` /
``geo_linearize`` / ``photo_residuals`` / ``geo_residuals`` and the
reference's own ``AlignmentProblem._accumulate`` (:615-628) on a recorder
in place of the dense n_vars^2 matrix.  The recorder captures every
``jtj[block] += value`` / ``grad[seg] += value`` the reference performs;
this process replays them in the reference's edge order into the real
matrix.  Because ``0.0 + v == v`` exactly, the replay produces the same bits
as the sequential reference: the normal equations, the PCG (the reference's
``pcg_solve`` on the reference's ``NormalEquations``), every record and the
final poses are those of a single-process reference run, which would take
~2 CPU-hours at cfg4.  The dense-edge list is the reference's own
(``build_dense_edges`` at the initial poses, tests/golden/edges_cfg*.npy,
checked here against the reference predicate on a sample of pairs).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from scanfuse import filters as RF  # noqa: E402
from scanfuse import frames as RFr  # noqa: E402
from scanfuse import geometry as RG  # noqa: E402
from scanfuse import solver as RS  # noqa: E402

from scenes import synth  # noqa: E402

N_WORK = int(os.environ.get("GOLDEN_WORKERS", os.cpu_count() or 8))

# name -> (synth config, SolverConfig overrides, dense-edge fixture or None)
VARIANTS = {
    "cfg4": ("cfg4", {}, "edges_cfg4.npy"),
    "cfg5": ("cfg5", {}, "edges_cfg5.npy"),
    "cfg2s": ("cfg2", {"dense_pixel_stride": 2}, None),
    "cfg2b": ("cfg2", {"dense_bidirectional": True}, None),
    "cfg3s": ("cfg3", {"dense_pixel_stride": 2}, None),
    "cfg3b": ("cfg3", {"dense_bidirectional": True}, None),
    "cfg3sb": ("cfg3", {"dense_pixel_stride": 3, "dense_bidirectional": True}, None),
}


class _Recorder:
    """Stands in for jtj / grad inside the reference's _accumulate."""

    def __init__(self, shape_of):
        self.ops = []
        self._shape_of = shape_of

    def __getitem__(self, key):
        return np.zeros(self._shape_of(key))

    def __setitem__(self, key, value):
        self.ops.append((key, np.array(value)))


def _seg(s):
    return s.stop - s.start


def ref_caches(scene):
    out = {}
    for f, c in scene.caches.items():
        k = c.intrinsics_low
        out[f] = RFr.CachedFrame(
            index=f, intensity_low=None, grad_low=c.grad_low, depth_low=None,
            points_low=c.points_low, normals_low=c.normals_low,
            intrinsics_low=RG.Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height),
            valid_depth=c.valid_depth, valid_normal=c.valid_normal)
    return out


def _poses_from(arr_R, arr_t, ids):
    return {f: RG.RigidTransform(arr_R[k], arr_t[k]) for k, f in enumerate(ids)}


def _worker(conn, ids, caches, frame_to_var, directed, mine):
    """Owns the directed edges ``mine`` (indices into ``directed``)."""
    photo, geo = {}, {}
    while True:
        msg = conn.recv()
        if msg[0] == "quit":
            return
        _, R, t, wp, wg, w_dense, cfg_kw, what = msg
        poses = _poses_from(R, t, ids)
        out = []
        if what == "lin":
            config = RS.SolverConfig(**cfg_kw)
            stride = config.dense_pixel_stride
            photo.clear()
            geo.clear()
            for e in mine:
                i, j = directed[e]
                ci, cj = caches[i], caches[j]
                vi, vj = frame_to_var[i], frame_to_var[j]
                rec = []
                if wp > 0.0:
                    a = RS.associate_photo(poses, i, j, ci, cj, stride)
                    photo[e] = a
                    if a.points.shape[0]:
                        res, Ji, Jj = RS.photo_linearize(poses, a, cj)
                        esum = float(np.sum(res ** 2))
                        jt, gr = _Recorder(lambda k: (_seg(k[0]), _seg(k[1]))), _Recorder(lambda k: (_seg(k),))
                        RS.AlignmentProblem._accumulate(jt, gr, Ji, Jj, res, vi, vj, w_dense * wp)
                        rec.append(("photo", esum, jt.ops, gr.ops, a.points.shape[0]))
                    else:
                        rec.append(("photo", None, [], [], 0))
                if wg > 0.0:
                    a = RS.associate_geo(poses, i, j, ci, cj, config, stride)
                    geo[e] = a
                    if a.points.shape[0]:
                        res, Ji, Jj = RS.geo_linearize(poses, a)
                        jt, gr = _Recorder(lambda k: (_seg(k[0]), _seg(k[1]))), _Recorder(lambda k: (_seg(k),))
                        RS.AlignmentProblem._accumulate(jt, gr, Ji[:, None, :], Jj[:, None, :], res[:, None],
                                                        vi, vj, w_dense * wg)
                        esum = float(np.sum(res ** 2))
                        rec.append(("geo", esum, jt.ops, gr.ops, a.points.shape[0]))
                    else:
                        rec.append(("geo", None, [], [], 0))
                out.append((e, rec))
        else:  # frozen energy
            for e in mine:
                ep = eg = None
                if e in photo:
                    a = photo[e]
                    ep = float(np.sum(RS.photo_residuals(poses, a, caches[a.frame_j]) ** 2))
                if e in geo:
                    eg = float(np.sum(RS.geo_residuals(poses, geo[e]) ** 2))
                out.append((e, ep, eg))
        conn.send(out)


class PooledProblem(RS.AlignmentProblem):
    """The reference AlignmentProblem with its per-edge loops on a pool."""

    def start(self, config):
        self.directed = list(RS._directed_edges(self.dense_edges, config.dense_bidirectional))
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        nw = max(1, min(N_WORK, len(self.directed)))
        for k in range(nw):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, self.frame_ids, self.caches, self.frame_to_var,
                                                  self.directed, list(range(k, len(self.directed), nw))))
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.trace_R, self.trace_t = [], []

    def stop(self):
        for c in self.conns:
            c.send(("quit",))
        for p in self.procs:
            p.join()

    def _broadcast(self, what, weights, w_dense, config):
        R = np.stack([np.asarray(self.poses[f].rotation) for f in self.frame_ids])
        t = np.stack([np.asarray(self.poses[f].translation) for f in self.frame_ids])
        kw = {k: getattr(config, k) for k in config.__dataclass_fields__}
        for c in self.conns:
            c.send((what, R, t, weights.photo, weights.geo, w_dense, kw, what))
        res = []
        for c in self.conns:
            res.extend(c.recv())
        res.sort(key=lambda r: r[0])
        return res

    def _dense_blocks(self, weights, w_dense, config):
        """solver.py:582-613 with the edge loop body on the pool, replayed in order."""
        self._last_cfg = config
        jtj = np.zeros((self.n_vars, self.n_vars))
        grad = np.zeros(self.n_vars)
        photo_assocs, geo_assocs = [], []
        energy_photo = 0.0
        energy_geo = 0.0
        for e, rec in self._broadcast("lin", weights, w_dense, config):
            for kind, esum, jops, gops, m in rec:
                (photo_assocs if kind == "photo" else geo_assocs).append((e, m))
                if esum is None:
                    continue
                # _accumulate order: for va: grad first, then the two jtj blocks
                gi = iter(gops)
                ji = iter(jops)
                if kind == "photo":
                    energy_photo += esum
                i, j = self.directed[e]
                for va in (self.frame_to_var[i], self.frame_to_var[j]):
                    if va < 0:
                        continue
                    key, val = next(gi)
                    grad[key] += val
                    for vb in (self.frame_to_var[i], self.frame_to_var[j]):
                        if vb < 0:
                            continue
                        key, val = next(ji)
                        jtj[key] += val
                if kind == "geo":
                    energy_geo += esum
        return jtj, grad, energy_photo, energy_geo, photo_assocs, geo_assocs

    def _energy_with_frozen_associations(self, weights, w_dense, photo_assocs, geo_assocs):
        """solver.py:662-672; the per-association sums come from the pool."""
        self.trace_R.append(np.stack([np.asarray(self.poses[f].rotation) for f in self.frame_ids]))
        self.trace_t.append(np.stack([np.asarray(self.poses[f].translation) for f in self.frame_ids]))
        _, energy = RS.eval_sparse(self.poses, self.corr_sets)
        energy *= weights.sparse
        if w_dense > 0.0:
            per = {e: (ep, eg) for e, ep, eg in self._broadcast("energy", weights, w_dense, self._last_cfg)}
            e_photo = sum(per[e][0] for e, _ in photo_assocs)
            e_geo = sum(per[e][1] for e, _ in geo_assocs)
            energy += w_dense * (weights.photo * e_photo + weights.geo * e_geo)
        return energy


def pose_arrays(poses, ids):
    return (np.stack([np.asarray(poses[f].rotation) for f in ids]),
            np.stack([np.asarray(poses[f].translation) for f in ids]))


def check_edges(ids, poses, caches, config, edges, n_sample=400, seed=5):
    """Spot-check the fixture edge list against the reference predicate."""
    rng = np.random.default_rng(seed)
    eset = set(edges)
    n = len(ids)
    for _ in range(n_sample):
        a, b = sorted(rng.choice(n, size=2, replace=False))
        i, j = ids[a], ids[b]
        ok = (RFr.view_angle_deg(poses[i], poses[j]) < config.view_angle_max_deg
              and RFr.frustum_overlap(caches[i], poses[i], caches[j], poses[j]) > 0.0
              and RFr.frustum_overlap(caches[j], poses[j], caches[i], poses[i]) > 0.0)
        assert ok == ((i, j) in eset), (i, j)


def solve_golden(name):
    cfg_name, overrides, edge_file = VARIANTS[name]
    t0 = time.time()
    scene = synth.make(cfg_name)
    ids = scene.frame_ids
    caches = ref_caches(scene)
    init = {f: RG.RigidTransform(np.array(p.rotation), np.array(p.translation)) for f, p in scene.init.items()}
    sets = [RF.CorrespondenceSet(s.frame_i, s.frame_j, s.points_i, s.points_j,
                                 np.zeros((len(s), 2), dtype=int), None, True) for s in scene.corr_sets]
    w = RS.EnergyWeights(**scene.weights)
    cfg = RS.SolverConfig(**{**scene.config, **overrides})
    if edge_file is not None:
        edges = [tuple(int(x) for x in e) for e in np.load(HERE / edge_file)]
        check_edges(ids, init, caches, cfg, edges)
    else:
        edges = RS.build_dense_edges(ids, init, caches, cfg)
    print(f"{name}: scene + edges {time.time() - t0:.0f} s, {len(edges)} edges", flush=True)

    orig = RS.build_dense_edges

    def fixture_edges(frame_ids, poses, cs, config):
        assert all(poses[f] is init[f] for f in frame_ids)  # solve() filters at the initial poses
        return list(edges)

    RS.build_dense_edges = fixture_edges
    try:
        prob = PooledProblem(ids, dict(init), sets, caches)
        prob.dense_edges = list(edges)
        prob.start(cfg)
        t1 = time.time()
        stats = prob.solve(w, cfg, scene.max_iterations)
        prob.stop()
    finally:
        RS.build_dense_edges = orig
    print(f"{name}: solve {time.time() - t1:.0f} s, {len(stats.iterations)} records", flush=True)
    fields = ("energy_before", "energy_after", "dense_weight", "pcg_iterations", "pcg_residual",
              "step_norm", "accepted")
    out = {
        "edges": np.array(edges, dtype=np.int64).reshape(-1, 2),
        "records": np.array([[float(getattr(r, f)) for f in fields] for r in stats.iterations]),
        "flags": np.array([stats.converged, stats.aborted]),
        "config_overrides": np.array(repr(overrides)),
        "trace_R": np.array(prob.trace_R), "trace_t": np.array(prob.trace_t),
    }
    out["final_R"], out["final_t"] = pose_arrays(prob.poses, ids)
    out["init_R"], out["init_t"] = pose_arrays(init, ids)
    np.savez_compressed(HERE / f"solve_{name}.npz", **out)
    for r in stats.iterations:
        print("  ", r, flush=True)
    print(f"{name}: done in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["cfg2s", "cfg2b", "cfg3s", "cfg3b"]:
        solve_golden(nm)
