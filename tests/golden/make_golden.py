"""Generate the golden vectors by running the UNMODIFIED reference solver.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [cfg1 cfg2 cfg3 units]

Inputs come from scenes.synth (deterministic); every output
(edge lists, linearisation snapshot, per-iteration records, final poses,
association sizes, Jacobians, overlaps) is produced by scanfuse 0.1.0 from
/root/reference/pkg/src.  The caches fed to the reference are built by the
reference's own build_cache and checked bit-identical to ours.
"""

from __future__ import annotations

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
from scipy import ndimage  # noqa: E402

from scenes import synth  # noqa: E402
from paper_1604_01093_b200.cache import RgbdFrame  # noqa: E402

K = RG.Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)


def ref_pose(p):
    return RG.RigidTransform(np.array(p.rotation, dtype=np.float64), np.array(p.translation, dtype=np.float64))


def ref_k(k):
    return RG.Intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height)


def ref_caches_from_renders(scene):
    out = {}
    kr = ref_k(scene.render_k)
    for f, (g, d) in scene.renders.items():
        fr = RFr.RgbdFrame(index=f, color=np.repeat(g[..., None], 3, axis=2), depth=d)
        out[f] = RFr.build_cache(fr, kr, scene.low_size[0], scene.low_size[1])
    return out


def ref_sets(sets):
    return [RF.CorrespondenceSet(frame_i=s.frame_i, frame_j=s.frame_j, points_i=s.points_i,
                                 points_j=s.points_j, indices=np.zeros((len(s), 2), dtype=int),
                                 transform=None, valid=True) for s in sets]


def pose_arrays(poses, ids):
    return (np.stack([np.asarray(poses[f].rotation) for f in ids]),
            np.stack([np.asarray(poses[f].translation) for f in ids]))


def same_planes(a, b) -> bool:
    for f in a:
        for n in ("valid_depth", "valid_normal", "points_low", "normals_low", "grad_low"):
            if not np.array_equal(getattr(a[f], n), getattr(b[f], n)):
                return False
    return True


def config_golden(name):
    scene = synth.make(name)
    ids = scene.frame_ids
    out = {"ids": np.array(ids)}
    out["init_R"], out["init_t"] = pose_arrays(scene.init, ids)
    out["truth_R"], out["truth_t"] = pose_arrays(scene.truth, ids)
    frames, off, pi, pj = [], [0], [], []
    for s in scene.corr_sets:
        frames.append((s.frame_i, s.frame_j))
        off.append(off[-1] + len(s))
        pi.append(s.points_i)
        pj.append(s.points_j)
    out["set_frames"] = np.array(frames, dtype=np.int64)
    out["set_off"] = np.array(off, dtype=np.int64)
    out["pts_i"] = np.vstack(pi)
    out["pts_j"] = np.vstack(pj)
    w = RS.EnergyWeights(**scene.weights)
    cfg = RS.SolverConfig(**scene.config)
    out["weights"] = np.array([w.sparse, w.photo, w.geo, w.dense_ramp[0], w.dense_ramp[1]], float)
    out["config"] = np.array([cfg.batch_iterations, cfg.pcg_max_iterations, cfg.pcg_tolerance,
                              cfg.pcg_restart_interval, cfg.min_relative_decrease,
                              cfg.view_angle_max_deg, cfg.geo_distance_max, cfg.geo_normal_min,
                              cfg.dense_pixel_stride, float(cfg.dense_bidirectional),
                              cfg.prune_residual_max], float)
    out["max_iterations"] = np.array(-1 if scene.max_iterations is None else scene.max_iterations)
    caches = None
    if scene.caches is not None:
        caches = ref_caches_from_renders(scene)
        assert same_planes(caches, scene.caches), "our build_cache differs from the reference's"
        out["cache_sha"] = np.array(synth.cache_digest(scene.caches))
        if name == "cfg2":  # 640x480 renders are large: keep the reduced planes
            fs = [caches[f] for f in ids]
            out["vd"] = np.stack([c.valid_depth for c in fs])
            out["vn"] = np.stack([c.valid_normal for c in fs])
            out["pts"] = np.stack([c.points_low for c in fs])
            out["nrm"] = np.stack([c.normals_low for c in fs])
            out["grad"] = np.stack([c.grad_low for c in fs])
            k = fs[0].intrinsics_low
            out["k_low"] = np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height], float)
        else:
            out["gray"] = np.stack([scene.renders[f][0] for f in ids])
            out["depth"] = np.stack([scene.renders[f][1] for f in ids])
            k = scene.render_k
            out["render_k"] = np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height], float)
            out["low_size"] = np.array(scene.low_size)
    init = {f: ref_pose(scene.init[f]) for f in ids}
    sets = ref_sets(scene.corr_sets)

    # pair filter
    t0 = time.time()
    if caches is not None:
        edges = RS.build_dense_edges(ids, init, caches, cfg)
        out["edges"] = np.array(edges, dtype=np.int64).reshape(-1, 2)
        print(f"{name}: {len(edges)} edges in {time.time() - t0:.1f}s", flush=True)
    # linearisation snapshot at the initial poses, dense weight 1
    prob = RS.AlignmentProblem(ids, init, sets, caches)
    w_d = 1.0 if caches is not None else 0.0
    if caches is not None:
        prob.dense_edges = edges
    eqs, energy, pa, ga = prob.normal_equations(w, w_d, cfg)
    rng = np.random.default_rng(99)
    u = rng.normal(size=eqs.n_vars)
    out["lin_energy"] = np.array(energy)
    out["lin_grad"] = eqs.gradient
    out["lin_diag"] = eqs.diagonal
    out["lin_u"] = u
    out["lin_Au"] = eqs.apply(u)
    x, info = RS.pcg_solve(eqs, cfg.pcg_max_iterations, cfg.pcg_tolerance, cfg.pcg_restart_interval)
    out["pcg_x"] = x
    out["pcg_info"] = np.array([info.iterations, info.relative_residual])
    out["photo_m"] = np.array([a.points.shape[0] for a in pa], dtype=np.int64)
    out["geo_m"] = np.array([a.points.shape[0] for a in ga], dtype=np.int64)
    prob._apply_step(x)
    out["frozen_energy"] = np.array(prob._energy_with_frozen_associations(w, w_d, pa, ga))
    # full solve from the initial poses
    t0 = time.time()
    prob = RS.AlignmentProblem(ids, init, sets, caches)
    stats = prob.solve(w, cfg, scene.max_iterations)
    print(f"{name}: solve {time.time() - t0:.1f}s, {len(stats.iterations)} records", flush=True)
    fields = ("energy_before", "energy_after", "dense_weight", "pcg_iterations", "pcg_residual",
              "step_norm", "accepted")
    out["records"] = np.array([[float(getattr(r, f)) for f in fields] for r in stats.iterations])
    out["flags"] = np.array([stats.converged, stats.aborted])
    out["final_R"], out["final_t"] = pose_arrays(prob.poses, ids)
    np.savez_compressed(HERE / f"{name}.npz", **out)


def textured_cache(index=0, seed=0, tilt=0.05):
    """test_solver.py:74-84 through the reference build_cache."""
    rng = np.random.default_rng(seed)
    noise = ndimage.gaussian_filter(rng.normal(size=(480, 640)), 8.0)
    noise = (noise - noise.min()) / (noise.max() - noise.min())
    color = np.repeat((40 + 170 * noise)[..., None].astype(np.uint8), 3, axis=2)
    xs = np.linspace(-1, 1, 640)[None, :]
    ys = np.linspace(-1, 1, 480)[:, None]
    depth = (2.0 + tilt * xs + 0.5 * tilt * ys).astype(np.float32)
    fr = RFr.RgbdFrame(index=index, color=color, depth=np.broadcast_to(depth, (480, 640)).copy())
    return RFr.build_cache(fr, K), color, fr.depth


def units_golden():
    out = {}
    # textured caches of test_solver.py (seed, tilt) and their colour/depth inputs
    specs = [(3, 0.05), (6, 0.05), (7, 0.05), (4, 0.0), (5, 0.0)]
    caches = {}
    for seed, tilt in specs:
        c, color, depth = textured_cache(0, seed, tilt)
        ours = synth.build_cache(RgbdFrame(0, color, depth), synth.K_FULL)
        assert same_planes({0: c}, {0: ours})
        caches[seed] = c
        out[f"tex{seed}_sha"] = np.array(synth.cache_digest({0: ours}))
    # photo / geo association + linearisation on random pose pairs (test_solver.py:173-230)
    rng = np.random.default_rng(8)
    cfg = RS.SolverConfig()
    for kind, seed in (("photo", 6), ("geo", 7)):
        cs = {0: caches[seed], 1: caches[seed]}
        for trial in range(5):
            rel = RG.exp_twist(RG.TwistParams(rng.normal(scale=0.01, size=3), rng.normal(scale=0.01, size=3)))
            base = RG.exp_twist(RG.TwistParams(rng.normal(scale=0.2, size=3), rng.normal(scale=0.2, size=3)))
            poses = {0: base, 1: base @ rel}
            key = f"{kind}{trial}"
            out[key + "_R"], out[key + "_t"] = pose_arrays(poses, [0, 1])
            # selection mask over source pixels, recomputed with the reference's
            # own geometry and checked against what associate_* returned
            c0, c1 = cs[0], cs[1]
            ys, xs = RS._source_pixel_data(c0, 1, kind == "geo")
            rel_ = poses[1].inverse() @ poses[0]
            warped = rel_.apply(c0.points_low[ys, xs].astype(np.float64))
            pix, front = c1.intrinsics_low.project_many(warped)
            if kind == "photo":
                a = RS.associate_photo(poses, 0, 1, c0, c1)
                res, Ji, _ = RS.photo_linearize(poses, a, c1)
                k1 = c1.intrinsics_low
                keep = (front & (pix[:, 0] >= 0) & (pix[:, 0] <= k1.width - 1)
                        & (pix[:, 1] >= 0) & (pix[:, 1] <= k1.height - 1))
                assert np.array_equal(c0.points_low[ys, xs][keep].astype(np.float64), a.points)
                res2 = RS.photo_residuals(poses, a, c1)
                tgt = np.zeros(0, dtype=np.int64)
            else:
                a = RS.associate_geo(poses, 0, 1, c0, c1, cfg)
                res, Ji, _ = RS.geo_linearize(poses, a)
                xi = np.clip(np.round(pix[:, 0]).astype(int), 0, 79)
                yi = np.clip(np.round(pix[:, 1]).astype(int), 0, 59)
                pts_all = c0.points_low[ys, xs].astype(np.float64)
                keep = np.zeros(ys.size, dtype=bool)
                rows = {tuple(p) for p in a.points}
                keep = np.array([tuple(p) in rows for p in pts_all])
                assert np.array_equal(pts_all[keep], a.points)
                tgt = (yi * 80 + xi)[keep]
                assert np.array_equal(c1.points_low.reshape(-1, 3)[tgt].astype(np.float64), a.targets)
                res2 = RS.geo_residuals(poses, a)
            mask = np.zeros(c0.valid_depth.shape, dtype=bool)
            mask[ys[keep], xs[keep]] = True
            out[key + "_mask"] = np.packbits(mask.ravel())
            out[key + "_tgt"] = tgt.astype(np.int32)
            dec = slice(None, None, 9)
            out[key + "_res"], out[key + "_J"], out[key + "_res2"] = res[dec], Ji[dec], res2[dec]
            out[key + "_sums"] = np.array([np.sum(res ** 2), np.sum(Ji ** 2), np.sum(res2 ** 2)])
    # frustum overlap (test_frames.py:81-101) on the flat make_frame cache
    fr = RFr.RgbdFrame(index=0, color=np.random.default_rng(1).integers(0, 255, size=(480, 640, 3), dtype=np.uint8),
                       depth=np.full((480, 640), 2.0, dtype=np.float32))
    flat = RFr.build_cache(fr, K)
    out["flat_sha"] = np.array(synth.cache_digest({0: flat}))
    eye = RG.RigidTransform.identity()
    flipped = RG.exp_twist(RG.TwistParams(np.array([0.0, np.pi, 0.0]), np.zeros(3)))
    vw = 80 * 2.0 / flat.intrinsics_low.fx
    shifted = RG.RigidTransform(np.eye(3), np.array([vw / 2, 0.0, 0.0]))
    out["overlap_flat"] = np.array([RFr.frustum_overlap(flat, eye, flat, eye),
                                    RFr.frustum_overlap(flat, eye, flat, flipped),
                                    RFr.frustum_overlap(flat, eye, flat, shifted),
                                    RFr.view_angle_deg(eye, flipped)])
    # random multi-frame filter problems on textured caches, incl. exact-boundary poses
    rng = np.random.default_rng(41)
    for trial in range(6):
        n = 9
        poses = {}
        for f in range(n):
            if trial == 0 and f < 4:
                # identical/axis-shifted poses: points land exactly on border pixel centres
                poses[f] = RG.RigidTransform(np.eye(3), np.array([0.5 * f * vw / 2 * (f % 2), 0.0, 0.0]))
            else:
                poses[f] = RG.exp_twist(RG.TwistParams(rng.normal(scale=0.5, size=3), rng.normal(scale=0.6, size=3)))
        cs = {f: (caches[(3, 6, 7, 4, 5)[f % 5]] if f % 3 else flat) for f in range(n)}
        edges = RS.build_dense_edges(list(range(n)), poses, cs, cfg)
        out[f"filt{trial}_R"], out[f"filt{trial}_t"] = pose_arrays(poses, list(range(n)))
        out[f"filt{trial}_edges"] = np.array(edges, dtype=np.int64).reshape(-1, 2)
        ov = [RFr.frustum_overlap(cs[a], poses[a], cs[b], poses[b]) for a in range(n) for b in range(n) if a != b]
        out[f"filt{trial}_overlap"] = np.array(ov)
        out[f"filt{trial}_angle"] = np.array([RFr.view_angle_deg(poses[a], poses[b]) for a in range(n) for b in range(n) if a != b])
    np.savez_compressed(HERE / "units.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["units", "cfg1", "cfg2", "cfg3"]
    for name in which:
        t0 = time.time()
        units_golden() if name == "units" else config_golden(name)
        print(f"{name} done in {time.time() - t0:.1f}s", flush=True)
