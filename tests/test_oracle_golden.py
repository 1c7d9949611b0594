"""Pin the CPU oracle (oracle/scanfuse_oracle.py) to the reference's golden vectors.

tests/golden/*.npz were produced by the unmodified reference solver
(tests/golden/make_golden.py).  These tests run without a GPU.
"""

import numpy as np
import pytest

from golden_io import GoldenScene, load, pose_errors
from oracle import scanfuse_oracle as O
from scenes import synth
from paper_1604_01093_b200.se3 import RigidTransform

FIELDS = ("energy_before", "energy_after", "dense_weight", "pcg_iterations", "pcg_residual",
          "step_norm", "accepted")


def _tuples(poses):
    return {f: O.pose_of(p) for f, p in poses.items()}


@pytest.fixture(scope="module", params=["cfg1", "cfg2", "cfg3"])
def scene(request):
    return GoldenScene(request.param)


def test_inputs_rebuild_bit_exact(scene):
    assert scene.cache_sha_ok


def test_oracle_dense_edges_match_reference(scene):
    if scene.caches is None:
        pytest.skip("sparse-only configuration")
    edges = O.dense_edges(scene.ids, _tuples(scene.init), scene.caches, scene.config["view_angle_max_deg"])
    assert np.array_equal(np.array(edges).reshape(-1, 2), scene.g["edges"])


def test_oracle_linearization_snapshot(scene):
    g = scene.g
    P = O.Problem(scene.ids, _tuples(scene.init), scene.corr_sets, scene.caches)
    wd = 0.0
    if scene.caches is not None:
        P.edges = [tuple(e) for e in g["edges"].tolist()]
        wd = 1.0
    S, energy, frozen = P.linearize(scene.weights, wd, scene.config)
    assert energy == pytest.approx(float(g["lin_energy"]), rel=1e-12)
    scale = np.abs(g["lin_grad"]).max()
    np.testing.assert_allclose(S.gradient, g["lin_grad"], rtol=0, atol=1e-10 * scale)
    np.testing.assert_allclose(S.diagonal, g["lin_diag"], rtol=1e-10, atol=1e-12 * g["lin_diag"].max())
    Au = S.apply(g["lin_u"])
    np.testing.assert_allclose(Au, g["lin_Au"], rtol=0, atol=1e-10 * np.abs(g["lin_Au"]).max())
    if scene.caches is not None:
        assert np.array_equal([p[2].shape[0] for p in frozen[0]], g["photo_m"])
        assert np.array_equal([p[2].shape[0] for p in frozen[1]], g["geo_m"])
    x, its, rel, bad = O.pcg(S, scene.config["pcg_max_iterations"], scene.config["pcg_tolerance"],
                             scene.config["pcg_restart_interval"])
    assert not bad and its == int(g["pcg_info"][0])
    np.testing.assert_allclose(x, g["pcg_x"], rtol=0, atol=1e-7 * np.abs(g["pcg_x"]).max())
    P.step(x)
    assert P.frozen_energy(scene.weights, wd, frozen) == pytest.approx(float(g["frozen_energy"]), rel=1e-9)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_oracle_full_solve(name):
    scene = GoldenScene(name)
    g = scene.g
    poses, recs, conv, abort, edges = O.solve(scene.ids, _tuples(scene.init), scene.corr_sets,
                                              scene.caches, scene.weights, scene.config,
                                              scene.max_iterations)
    assert [conv, abort] == list(g["flags"])
    assert len(recs) == g["records"].shape[0]
    for r, ref in zip(recs, g["records"]):
        assert r["pcg_iterations"] == int(ref[3])
        assert r["accepted"] == bool(ref[6])
        assert r["energy_after"] == pytest.approx(ref[1], rel=1e-8)
    final = {f: RigidTransform(*poses[f]) for f in scene.ids}
    ref_final = {f: RigidTransform(g["final_R"][k], g["final_t"][k]) for k, f in enumerate(scene.ids)}
    re, te = pose_errors(final, ref_final)
    assert re < 1e-9 and te < 1e-9


def test_units_oracle_associations():
    u = load("units")
    from paper_1604_01093_b200.cache import RgbdFrame
    from scipy import ndimage

    def tex(seed, tilt=0.05):
        rng = np.random.default_rng(seed)
        noise = ndimage.gaussian_filter(rng.normal(size=(480, 640)), 8.0)
        noise = (noise - noise.min()) / (noise.max() - noise.min())
        color = np.repeat((40 + 170 * noise)[..., None].astype(np.uint8), 3, axis=2)
        xs = np.linspace(-1, 1, 640)[None, :]
        ys = np.linspace(-1, 1, 480)[:, None]
        depth = (2.0 + tilt * xs + 0.5 * tilt * ys).astype(np.float32)
        c = synth.build_cache(RgbdFrame(0, color, np.broadcast_to(depth, (480, 640)).copy()), synth.K_FULL)
        assert synth.cache_digest({0: c}) == str(u[f"tex{seed}_sha"])
        return c

    for kind, seed in (("photo", 6), ("geo", 7)):
        c = tex(seed)
        for trial in range(5):
            key = f"{kind}{trial}"
            poses = {0: (u[key + "_R"][0], u[key + "_t"][0]), 1: (u[key + "_R"][1], u[key + "_t"][1])}
            mask = np.unpackbits(u[key + "_mask"])[:4800].astype(bool).reshape(60, 80)
            if kind == "photo":
                pts, ref = O.assoc_photo(poses, 0, 1, c, c)
                res, J = O.photo_lin(poses, 0, 1, pts, ref, c)
                res2 = O.photo_res(poses, 0, 1, pts, ref, c)
            else:
                pts, nrm, tgt = O.assoc_geo(poses, 0, 1, c, c)
                res, J = O.geo_lin(poses, 0, 1, pts, nrm, tgt)
                res2 = O.geo_res(poses, 0, 1, pts, nrm, tgt)
            ys, xs = np.nonzero(mask)
            assert np.array_equal(pts, c.points_low[ys, xs].astype(np.float64))
            sums = u[key + "_sums"]
            assert np.sum(res ** 2) == pytest.approx(sums[0], rel=1e-10)
            assert np.sum(J ** 2) == pytest.approx(sums[1], rel=1e-10)
            assert np.sum(res2 ** 2) == pytest.approx(sums[2], rel=1e-10)
            np.testing.assert_allclose(J[::9], u[key + "_J"], rtol=1e-9, atol=1e-12)


def test_oracle_dense_verify_matches_reference_golden():
    """oracle.dense_verify == scanfuse.filters.dense_verify on every golden
    pair (tests/golden/make_verify_golden.py): counts, pass flags and the mean
    errors bit-for-bit."""
    from oracle import scanfuse_oracle as O
    from scenes import synth
    sc = synth.make("cfg3")
    g = load("verify")
    for k, (a, b) in enumerate(g["pairs"]):
        R = g["R"][k]
        R = np.asfortranarray(R) if g["f_order"][k] else np.ascontiguousarray(R)
        passed, e1, e2, n1, n2 = O.dense_verify(sc.caches[int(a)], sc.caches[int(b)], (R, g["t"][k]))
        assert passed == bool(g["passed"][k])
        assert (n1, n2) == (int(g["count_ij"][k]), int(g["count_ji"][k]))
        assert e1 == g["err_ij"][k] and e2 == g["err_ji"][k]


def test_host_build_cache_matches_reference_digests():
    """The scene generator's NumPy build_cache (scenes/host_cache.py, also the
    GPU test's diagnostic) is bit-identical to scanfuse.frames.build_cache on
    every golden input (tests/golden/make_cache_golden.py)."""
    import json
    import sys as _sys
    from golden_io import GOLDEN
    _sys.path.insert(0, str(GOLDEN))
    from make_cache_golden import PLANES, cache_inputs, digest
    from paper_1604_01093_b200 import cache as CA
    from paper_1604_01093_b200 import se3
    from scenes.host_cache import build_cache
    g = json.loads((GOLDEN / "cache_digests.json").read_text())
    for name, col, dep, (lw, lh), kk in cache_inputs():
        c = build_cache(CA.RgbdFrame(0, col, dep), se3.Intrinsics(*kk), lw, lh)
        for p in PLANES:
            assert digest(getattr(c, p)) == g[name][p], (name, p)


def test_oracle_tsdf_matches_reference_digests():
    """oracle.TsdfOracle == scanfuse.tsdf.TsdfVolume on the golden scenarios
    (tests/golden/make_tsdf_golden.py), except the slow 4 mm one."""
    import json
    import sys as _sys
    from golden_io import GOLDEN
    _sys.path.insert(0, str(GOLDEN))
    from make_tsdf_golden import SCENARIOS, tsdf_inputs, volume_digest
    from paper_1604_01093_b200 import se3
    g = json.loads((GOLDEN / "tsdf_digests.json").read_text())
    frames, K, truth, noisy = tsdf_inputs()
    k = se3.Intrinsics(*K)
    for name, (vs, trunc, dw, steps) in SCENARIOS.items():
        if name == "vs04":
            continue
        o = O.TsdfOracle(vs, trunc, dw)
        for step, (fi, sign, nz) in enumerate(steps):
            err = None
            try:
                o.apply_frame(frames[fi][0], frames[fi][1], k, (noisy if nz else truth)[fi], sign)
            except ValueError as e:
                err = str(e)
            d = volume_digest(list(o.blocks), {c: tuple(b) for c, b in o.blocks.items()})
            exp = g[name][step]
            for key in ("blocks", "occupied", "data", "order"):
                assert d[key] == exp[key], (name, step, key)
            assert (err is None) == (exp["error"] is None)
