"""Load tests/golden/*.npz (made by tests/golden/make_golden.py from the reference)."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from scenes import synth
from paper_1604_01093_b200.cache import CachedFrame, CorrespondenceSet
from paper_1604_01093_b200.se3 import Intrinsics, RigidTransform

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def poses_from(R, t, ids):
    return {f: RigidTransform(np.array(R[k]), np.array(t[k])) for k, f in enumerate(ids)}


class GoldenScene:
    def __init__(self, name: str):
        g = load(name)
        self.g = g
        self.name = name
        self.ids = [int(x) for x in g["ids"]]
        self.init = poses_from(g["init_R"], g["init_t"], self.ids)
        self.truth = poses_from(g["truth_R"], g["truth_t"], self.ids)
        off = g["set_off"]
        self.corr_sets = [
            CorrespondenceSet(int(a), int(b), g["pts_i"][off[k]:off[k + 1]], g["pts_j"][off[k]:off[k + 1]],
                              np.zeros((off[k + 1] - off[k], 2), dtype=int), None, True)
            for k, (a, b) in enumerate(g["set_frames"])]
        w = g["weights"]
        self.weights = dict(sparse=w[0], photo=w[1], geo=w[2], dense_ramp=(int(w[3]), int(w[4])))
        c = g["config"]
        self.config = dict(batch_iterations=int(c[0]), pcg_max_iterations=int(c[1]),
                           pcg_tolerance=c[2], pcg_restart_interval=int(c[3]),
                           min_relative_decrease=c[4], view_angle_max_deg=c[5],
                           geo_distance_max=c[6], geo_normal_min=c[7],
                           dense_pixel_stride=int(c[8]), dense_bidirectional=bool(c[9]),
                           prune_residual_max=c[10])
        mi = int(g["max_iterations"])
        self.max_iterations = None if mi < 0 else mi
        self.caches = None
        if "vd" in g:
            k = g["k_low"]
            kl = Intrinsics(k[0], k[1], k[2], k[3], int(k[4]), int(k[5]))
            self.caches = {f: CachedFrame(f, None, g["grad"][i], None, g["pts"][i], g["nrm"][i], kl,
                                          g["vd"][i], g["vn"][i]) for i, f in enumerate(self.ids)}
        elif "gray" in g:
            k = g["render_k"]
            kr = Intrinsics(k[0], k[1], k[2], k[3], int(k[4]), int(k[5]))
            renders = {f: (g["gray"][i], g["depth"][i]) for i, f in enumerate(self.ids)}
            self.caches = synth.caches_from_renders(renders, kr, tuple(int(x) for x in g["low_size"]))
        if self.caches is not None and "cache_sha" in g:
            self.cache_sha_ok = synth.cache_digest(self.caches) == str(g["cache_sha"])
        else:
            self.cache_sha_ok = True

    def weights_obj(self, mod):
        return mod.EnergyWeights(**self.weights)

    def config_obj(self, mod):
        return mod.SolverConfig(**self.config)


def rot_err(Ra, Rb) -> float:
    """Angle of Ra^T Rb via atan2 (accurate for tiny angles)."""
    M = Ra.T @ Rb
    s = 0.5 * np.linalg.norm([M[2, 1] - M[1, 2], M[0, 2] - M[2, 0], M[1, 0] - M[0, 1]])
    c = 0.5 * (np.trace(M) - 1.0)
    return float(np.arctan2(s, c))


def pose_errors(pa: dict, pb: dict):
    """(max rotation angle error rad, max translation error m)."""
    re = max(rot_err(np.asarray(pa[f].rotation), np.asarray(pb[f].rotation)) for f in pa)
    te = max(float(np.linalg.norm(np.asarray(pa[f].translation) - np.asarray(pb[f].translation)))
             for f in pa)
    return re, te
