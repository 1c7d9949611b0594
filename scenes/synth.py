"""Deterministic synthetic workloads for the five BASELINE.json configurations.

There is no dataset in this environment, so every configuration is rendered
here:

* cfg1  11-frame chunk, sparse only: the reference's own test generator
        (`chunk_ground_truth` / `chunk_corr_sets`, test_solver.py:46-71) with
        seed 16, 4 GN x 10 PCG.
* cfg2  11 frames in a textured box room, rendered at 640x480 and reduced by
        `build_cache` to 80x60, sparse + dense, 4 GN x 10 PCG.
* cfg3-5 a facade "out-and-back" scan (bounded dense degree ~60 with loop
        closures) rendered directly at 80x60 (cfg3: 100 keyframes, cfg5:
        2000) or 160x120 (cfg4: 500), default weights and config.

Depth is the z-depth of a ray cast to the inside of an axis-aligned box;
colour is a 12-sinusoid procedural texture of the hit point.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_1604_01093_b200.cache import CachedFrame, CorrespondenceSet, RgbdFrame
from paper_1604_01093_b200.se3 import Intrinsics, RigidTransform, TwistParams, exp_twist

from .host_cache import build_cache

K_FULL = Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)


@dataclass
class Scene:
    name: str
    frame_ids: list
    truth: dict
    init: dict
    corr_sets: list
    caches: dict | None
    weights: dict = field(default_factory=dict)   # EnergyWeights kwargs
    config: dict = field(default_factory=dict)    # SolverConfig kwargs
    max_iterations: int | None = None
    renders: dict | None = None                   # frame -> (gray uint8, depth f32)
    render_k: Intrinsics | None = None
    low_size: tuple | None = None                 # (w, h) of the caches


# ---------------------------------------------------------------------------
# cfg1: the reference test generator, same RNG call sequence


def make_corr_set(frame_i, frame_j, points_i, points_j) -> CorrespondenceSet:
    n = len(points_i)
    return CorrespondenceSet(frame_i, frame_j, np.asarray(points_i, float),
                             np.asarray(points_j, float), np.zeros((n, 2), dtype=int), None, True)


def chunk_ground_truth(rng, n_frames=11, n_world=120, motion=0.03):
    poses = [RigidTransform.identity()]
    for _ in range(n_frames - 1):
        w = rng.normal(scale=motion, size=3) * 0.3
        v = rng.normal(scale=motion, size=3)
        poses.append(poses[-1] @ exp_twist(TwistParams(w, v)))
    world = rng.uniform([-1.5, -1.2, 1.0], [1.5, 1.2, 3.5], size=(n_world, 3))
    return poses, world


def chunk_corr_sets(rng, poses, world, per_pair=25, noise=0.0):
    out = []
    n = len(poses)
    for i in range(n):
        inv_i = poses[i].inverse()
        for j in range(i + 1, n):
            inv_j = poses[j].inverse()
            pick = rng.choice(world.shape[0], size=per_pair, replace=False)
            a = inv_i.apply(world[pick])
            b = inv_j.apply(world[pick])
            if noise > 0.0:
                a = a + rng.normal(scale=noise, size=a.shape)
                b = b + rng.normal(scale=noise, size=b.shape)
            out.append(make_corr_set(i, j, a, b))
    return out


def config1() -> Scene:
    rng = np.random.default_rng(16)
    truth, world = chunk_ground_truth(rng)
    sets = chunk_corr_sets(rng, truth, world)
    ids = list(range(11))
    return Scene("cfg1", ids, dict(enumerate(truth)),
                 {i: RigidTransform.identity() for i in ids}, sets, None,
                 weights=dict(sparse=1.0, photo=0.0, geo=0.0),
                 config=dict(pcg_max_iterations=10), max_iterations=4)


# ---------------------------------------------------------------------------
# box renderer


class BoxWorld:
    def __init__(self, lo, hi, seed=1234):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        rng = np.random.default_rng(seed)
        self.freq = rng.normal(0.0, 6.0, size=(12, 3))
        self.phase = rng.uniform(0.0, 2.0 * np.pi, size=12)

    def render(self, pose: RigidTransform, k: Intrinsics):
        """(gray uint8 (h,w), depth float32 (h,w)) seen from `pose`."""
        xs, ys = np.meshgrid(np.arange(k.width, dtype=np.float64),
                             np.arange(k.height, dtype=np.float64))
        dc = np.stack([(xs - k.cx) / k.fx, (ys - k.cy) / k.fy, np.ones_like(xs)], axis=-1)
        dw = dc @ np.asarray(pose.rotation).T
        o = np.asarray(pose.translation, dtype=np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            t_hi = (self.hi - o) / dw
            t_lo = (self.lo - o) / dw
        t_axis = np.where(dw > 0, t_hi, np.where(dw < 0, t_lo, np.inf))
        s = np.min(t_axis, axis=-1)
        hit = o + s[..., None] * dw
        tex = np.mean(np.sin(hit @ self.freq.T + self.phase), axis=-1)
        gray = (40.0 + 190.0 * np.clip(0.5 + 0.45 * tex, 0.0, 1.0)).astype(np.uint8)
        depth = s.astype(np.float32)
        depth[~np.isfinite(depth) | (depth <= 0)] = 0.0
        return gray, depth


def _cache_from_render(index, gray, depth, k_render, low_w, low_h) -> CachedFrame:
    color = np.repeat(gray[..., None], 3, axis=2)
    return build_cache(RgbdFrame(index, color, depth), k_render, low_w, low_h)


def _perturb(rng, pose, rot_sigma, trans_sigma):
    return exp_twist(TwistParams(rng.normal(0.0, rot_sigma, 3), rng.normal(0.0, trans_sigma, 3))) @ pose


def _sparse_sets_by_sampling(rng, ids, truth, caches, samples=64, per_pair=25, min_keep=5,
                             noise=0.0, all_pairs=False):
    """Correspondences from truth reprojection of sampled valid pixels."""
    n = len(ids)
    Rs = np.stack([np.asarray(truth[f].rotation) for f in ids])
    ts = np.stack([np.asarray(truth[f].translation) for f in ids])
    samp_cam, samp_world = [], []
    for f in ids:
        c = caches[f]
        ys, xs = np.nonzero(c.valid_depth)
        pick = rng.choice(ys.size, size=min(samples, ys.size), replace=False)
        p = c.points_low[ys[pick], xs[pick]].astype(np.float64)
        samp_cam.append(p)
        samp_world.append(p @ np.asarray(truth[f].rotation).T + np.asarray(truth[f].translation))
    sets = []
    for a in range(n):
        wa = samp_world[a]
        # into every camera at once: q = R_b^T (w - t_b)
        q = np.einsum("bji,bmj->bmi", Rs, wa[None, :, :] - ts[:, None, :])
        k = caches[ids[a]].intrinsics_low
        z = q[..., 2]
        front = z > 1e-6
        zs = np.where(front, z, 1.0)
        u = k.fx * q[..., 0] / zs + k.cx
        v = k.fy * q[..., 1] / zs + k.cy
        inside = front & (u >= 0) & (u <= k.width - 1) & (v >= 0) & (v <= k.height - 1)
        for b in range(a + 1, n):
            sel = np.nonzero(inside[b])[0] if not all_pairs else np.arange(wa.shape[0])
            if sel.size < (min_keep if not all_pairs else 1):
                continue
            sel = sel[:per_pair]
            pa = samp_cam[a][sel]
            pb = q[b, sel]
            if noise > 0.0:
                pa = pa + rng.normal(0.0, noise, pa.shape)
                pb = pb + rng.normal(0.0, noise, pb.shape)
            sets.append(make_corr_set(ids[a], ids[b], pa, pb))
    return sets


def config2() -> Scene:
    rng = np.random.default_rng(2)
    world = BoxWorld((-4.0, -1.5, -4.0), (4.0, 1.5, 4.0))
    ids = list(range(11))
    truth = {0: RigidTransform.identity()}
    pose = truth[0]
    for f in ids[1:]:
        step = exp_twist(TwistParams(rng.normal(0.0, 0.02, 3) * np.array([0.3, 1.0, 0.3]),
                                     rng.normal(0.0, 0.03, 3)))
        pose = step @ pose
        pose = RigidTransform(pose.rotation, np.clip(pose.translation, world.lo + 1.0, world.hi - 1.0))
        truth[f] = pose
    caches, renders = {}, {}
    for f in ids:
        gray, depth = world.render(truth[f], K_FULL)
        renders[f] = (gray, depth)
        caches[f] = _cache_from_render(f, gray, depth, K_FULL, 80, 60)
    sets = _sparse_sets_by_sampling(rng, ids, truth, caches, samples=200, per_pair=25)
    init = {0: truth[0]}
    for f in ids[1:]:
        init[f] = _perturb(rng, truth[f], 0.01, 0.02)
    return Scene("cfg2", ids, truth, init, sets, caches,
                 config=dict(pcg_max_iterations=10), max_iterations=4,
                 renders=renders, render_k=K_FULL, low_size=(80, 60))


def facade(n_frames: int, low_w: int, low_h: int, seed: int = 3, name: str = "facade") -> Scene:
    rng = np.random.default_rng(seed)
    half = (n_frames + 1) // 2
    world = BoxWorld((-3.0, -1.5, -1.0), (0.2 * half + 3.0, 1.5, 2.5))
    k_low = K_FULL.scaled(low_w, low_h)
    ids = list(range(n_frames))
    truth = {}
    for kf in ids:
        back = kf >= half
        s = (n_frames - 1 - kf) if back else kf
        t = np.array([0.2 * s + rng.normal(0.0, 0.02), rng.normal(0.0, 0.05),
                      (0.4 if back else 0.0) + rng.normal(0.0, 0.02)])
        w = np.array([rng.normal(0.0, 0.03), 0.35 * np.sin(kf / 7.0), rng.normal(0.0, 0.03)])
        truth[kf] = RigidTransform(exp_twist(TwistParams(w, np.zeros(3))).rotation, t)
    caches, renders = {}, {}
    for f in ids:
        gray, depth = world.render(truth[f], k_low)
        renders[f] = (gray, depth)
        caches[f] = _cache_from_render(f, gray, depth, k_low, low_w, low_h)
    sets = _sparse_sets_by_sampling(rng, ids, truth, caches, samples=64, per_pair=25,
                                    noise=0.002)
    init = {0: truth[0]}
    for f in ids[1:]:
        init[f] = _perturb(rng, truth[f], 0.01, 0.02)
    return Scene(name, ids, truth, init, sets, caches, renders=renders, render_k=k_low,
                 low_size=(low_w, low_h))


def caches_from_renders(renders: dict, render_k: Intrinsics, low_size) -> dict:
    """Rebuild the caches of a stored scene (tests/golden) from its renders."""
    return {f: _cache_from_render(f, g, d, render_k, low_size[0], low_size[1])
            for f, (g, d) in renders.items()}


def cache_digest(caches: dict) -> str:
    """sha256 over every solver-visible plane, frames in key order."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(caches):
        c = caches[f]
        for a in (c.valid_depth, c.valid_normal, c.points_low, c.normals_low, c.grad_low):
            h.update(np.ascontiguousarray(a).tobytes())
        k = c.intrinsics_low
        h.update(np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height], dtype=np.float64).tobytes())
    return h.hexdigest()


def config3() -> Scene:
    return facade(100, 80, 60, name="cfg3")


def config4() -> Scene:
    return facade(500, 160, 120, name="cfg4")


def config5() -> Scene:
    return facade(2000, 80, 60, name="cfg5")


CONFIGS = {"cfg1": config1, "cfg2": config2, "cfg3": config3, "cfg4": config4, "cfg5": config5}


def make(name: str) -> Scene:
    return CONFIGS[name]()
