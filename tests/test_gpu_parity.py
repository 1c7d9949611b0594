"""GPU parity: the drop-in (libsfb.so through the C ABI) against the reference's
golden vectors and the CPU oracle.

Tolerances (north star): poses 1e-4 rad / 1e-4 m, final energy 1e-5
relative, frame-pair filter bit-exact.  Intermediate quantities are held to
much tighter bounds than that (reordering-level, ~1e-9 relative).
"""

import numpy as np
import pytest

from golden_io import GoldenScene, load, pose_errors
from paper_1604_01093_b200 import solver as S
from scenes import synth
from paper_1604_01093_b200.cache import RgbdFrame
from paper_1604_01093_b200.se3 import RigidTransform

pytestmark = pytest.mark.gpu

POSE_TOL = 1e-4
ENERGY_RTOL = 1e-5


@pytest.fixture(scope="module")
def units():
    return load("units")


def _tex(seed, tilt=0.05):
    from scipy import ndimage
    rng = np.random.default_rng(seed)
    noise = ndimage.gaussian_filter(rng.normal(size=(480, 640)), 8.0)
    noise = (noise - noise.min()) / (noise.max() - noise.min())
    color = np.repeat((40 + 170 * noise)[..., None].astype(np.uint8), 3, axis=2)
    xs = np.linspace(-1, 1, 640)[None, :]
    ys = np.linspace(-1, 1, 480)[:, None]
    depth = (2.0 + tilt * xs + 0.5 * tilt * ys).astype(np.float32)
    return synth.build_cache(RgbdFrame(0, color, np.broadcast_to(depth, (480, 640)).copy()), synth.K_FULL)


@pytest.fixture(scope="module")
def tex_caches(units):
    out = {}
    for seed, tilt in ((3, 0.05), (6, 0.05), (7, 0.05), (4, 0.0), (5, 0.0)):
        c = _tex(seed, tilt)
        assert synth.cache_digest({0: c}) == str(units[f"tex{seed}_sha"])
        out[seed] = c
    return out


@pytest.fixture(scope="module")
def flat_cache(units):
    color = np.random.default_rng(1).integers(0, 255, size=(480, 640, 3), dtype=np.uint8)
    c = synth.build_cache(RgbdFrame(0, color, np.full((480, 640), 2.0, dtype=np.float32)), synth.K_FULL)
    assert synth.cache_digest({0: c}) == str(units["flat_sha"])
    return c


def _poses(R, t):
    return {k: RigidTransform(np.array(R[k]), np.array(t[k])) for k in range(R.shape[0])}


# ---------------------------------------------------------------- associations
@pytest.mark.parametrize("trial", range(5))
def test_photo_association_and_jacobian(units, tex_caches, trial):
    c = tex_caches[6]
    key = f"photo{trial}"
    poses = _poses(units[key + "_R"], units[key + "_t"])
    a = S.associate_photo(poses, 0, 1, c, c)
    mask = np.unpackbits(units[key + "_mask"])[:4800].astype(bool).reshape(60, 80)
    ys, xs = np.nonzero(mask)
    assert np.array_equal(a.points, c.points_low[ys, xs].astype(np.float64))  # bit-exact subset
    res, Ji, Jj = S.photo_linearize(poses, a, c)
    assert np.array_equal(Jj, -Ji)
    np.testing.assert_allclose(res[::9], units[key + "_res"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(Ji[::9], units[key + "_J"], rtol=1e-8, atol=1e-10)
    res2 = S.photo_residuals(poses, a, c)
    np.testing.assert_allclose(res2[::9], units[key + "_res2"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("trial", range(5))
def test_geo_association_and_jacobian(units, tex_caches, trial):
    c = tex_caches[7]
    key = f"geo{trial}"
    poses = _poses(units[key + "_R"], units[key + "_t"])
    a = S.associate_geo(poses, 0, 1, c, c, S.SolverConfig())
    mask = np.unpackbits(units[key + "_mask"])[:4800].astype(bool).reshape(60, 80)
    ys, xs = np.nonzero(mask)
    assert np.array_equal(a.points, c.points_low[ys, xs].astype(np.float64))
    tg = units[key + "_tgt"]
    assert np.array_equal(a.targets, c.points_low.reshape(-1, 3)[tg].astype(np.float64))
    res, Ji, Jj = S.geo_linearize(poses, a)
    np.testing.assert_allclose(res[::9], units[key + "_res"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(Ji[::9], units[key + "_J"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(S.geo_residuals(poses, a)[::9], units[key + "_res2"], rtol=1e-8, atol=1e-12)


# ---------------------------------------------------------------- pair filter
@pytest.mark.parametrize("trial", range(6))
def test_pair_filter_bit_exact(units, tex_caches, flat_cache, trial):
    n = 9
    poses = _poses(units[f"filt{trial}_R"], units[f"filt{trial}_t"])
    cs = {f: (tex_caches[(3, 6, 7, 4, 5)[f % 5]] if f % 3 else flat_cache) for f in range(n)}
    edges = S.build_dense_edges(list(range(n)), poses, cs, S.SolverConfig())
    assert np.array_equal(np.array(edges, dtype=np.int64).reshape(-1, 2), units[f"filt{trial}_edges"])
    from paper_1604_01093_b200.device_problem import DeviceProblem
    dp = DeviceProblem(n, [cs[f] for f in range(n)])
    dp.set_poses([poses[f] for f in range(n)])
    pairs = [(a, b) for a in range(n) for b in range(n) if a != b]
    ov = dp.frustum_overlap(pairs)
    assert np.array_equal(ov, units[f"filt{trial}_overlap"])  # exact fractions


def test_frustum_overlap_reference_cases(units, flat_cache):
    from paper_1604_01093_b200.device_problem import DeviceProblem
    from paper_1604_01093_b200.se3 import TwistParams, exp_twist
    eye = RigidTransform.identity()
    flipped = exp_twist(TwistParams(np.array([0.0, np.pi, 0.0]), np.zeros(3)))
    vw = 80 * 2.0 / flat_cache.intrinsics_low.fx
    shifted = RigidTransform(np.eye(3), np.array([vw / 2, 0.0, 0.0]))
    got = []
    for other in (eye, flipped, shifted):
        dp = DeviceProblem(2, [flat_cache, flat_cache])
        dp.set_poses([eye, other])
        got.append(dp.frustum_overlap([(0, 1)])[0])
    assert got == list(units["overlap_flat"][:3])
    assert got[0] == 1.0 and got[1] == 0.0 and abs(got[2] - 0.5) < 0.1


# ---------------------------------------------------------------- configurations
@pytest.fixture(scope="module", params=["cfg1", "cfg2", "cfg3"])
def scene(request):
    s = GoldenScene(request.param)
    assert s.cache_sha_ok, "synthetic inputs did not rebuild bit-exactly on this host"
    return s


def test_dense_edges_bit_exact(scene):
    if scene.caches is None:
        pytest.skip("sparse only")
    edges = S.build_dense_edges(scene.ids, scene.init, scene.caches, scene.config_obj(S))
    assert np.array_equal(np.array(edges, dtype=np.int64).reshape(-1, 2), scene.g["edges"])


def test_linearization_snapshot(scene):
    g = scene.g
    p = S.AlignmentProblem(scene.ids, scene.init, scene.corr_sets, scene.caches)
    wd = 0.0
    if scene.caches is not None:
        p.dense_edges = [tuple(e) for e in g["edges"].tolist()]
        wd = 1.0
    w, cfg = scene.weights_obj(S), scene.config_obj(S)
    eqs, energy, pa, ga = p.normal_equations(w, wd, cfg)
    assert energy == pytest.approx(float(g["lin_energy"]), rel=1e-10)
    gs = np.abs(g["lin_grad"]).max()
    np.testing.assert_allclose(eqs.gradient, g["lin_grad"], rtol=0, atol=1e-9 * gs)
    np.testing.assert_allclose(eqs.diagonal, g["lin_diag"], rtol=1e-9)
    Au = eqs.apply(g["lin_u"])
    np.testing.assert_allclose(Au, g["lin_Au"], rtol=0, atol=1e-9 * np.abs(g["lin_Au"]).max())
    if scene.caches is not None:
        assert [a.points.shape[0] for a in pa] == list(g["photo_m"])
        assert [a.points.shape[0] for a in ga] == list(g["geo_m"])
    x, info = S.pcg_solve(eqs, cfg.pcg_max_iterations, cfg.pcg_tolerance, cfg.pcg_restart_interval)
    assert info.iterations == int(g["pcg_info"][0])
    assert info.relative_residual == pytest.approx(g["pcg_info"][1], rel=1e-6)
    np.testing.assert_allclose(x, g["pcg_x"], rtol=0, atol=1e-7 * np.abs(g["pcg_x"]).max())


def test_full_solve_parity(scene):
    g = scene.g
    p = S.AlignmentProblem(scene.ids, scene.init, scene.corr_sets, scene.caches)
    stats = p.solve(scene.weights_obj(S), scene.config_obj(S), scene.max_iterations)
    assert [stats.converged, stats.aborted] == [bool(x) for x in g["flags"]]
    recs = g["records"]
    assert len(stats.iterations) == recs.shape[0]
    for r, ref in zip(stats.iterations, recs):
        assert r.pcg_iterations == int(ref[3])
        assert r.accepted == bool(ref[6])
        assert r.dense_weight == ref[2]
        assert r.energy_before == pytest.approx(ref[0], rel=ENERGY_RTOL)
        assert r.energy_after == pytest.approx(ref[1], rel=ENERGY_RTOL)
    assert stats.final_energy == pytest.approx(recs[-1][1], rel=ENERGY_RTOL)
    ref_final = {f: RigidTransform(g["final_R"][k], g["final_t"][k]) for k, f in enumerate(scene.ids)}
    re, te = pose_errors(p.poses, ref_final)
    assert re < POSE_TOL and te < POSE_TOL, (re, te)


def test_solve_is_bit_reproducible():
    s = GoldenScene("cfg2")
    out = []
    for _ in range(2):
        p = S.AlignmentProblem(s.ids, s.init, s.corr_sets, s.caches)
        st = p.solve(s.weights_obj(S), s.config_obj(S), s.max_iterations)
        out.append((np.stack([p.poses[f].rotation for f in s.ids]),
                    [r.energy_after for r in st.iterations]))
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]


def test_overlapped_setup_matches_direct_setup():
    """cfg3 (> 256 sets) builds the sparse problem while the frames upload
    (sfb_problem_attach_frames); the direct construction with the slots must
    give the bit-identical solve, and attaching twice is an error."""
    from paper_1604_01093_b200.device_problem import DeviceProblem
    from paper_1604_01093_b200.runtime import runtime
    s = GoldenScene("cfg3")
    assert len(s.corr_sets) > 256
    W, C = s.weights_obj(S), s.config_obj(S)
    p1 = S.AlignmentProblem(s.ids, s.init, s.corr_sets, s.caches)
    st1 = p1.solve(W, C, 3)
    p2 = S.AlignmentProblem(s.ids, s.init, s.corr_sets, s.caches)
    index = {f: k for k, f in enumerate(s.ids)}
    cl = [s.caches[f] for f in s.ids]
    frames, off, pi, pj = S._set_layout(s.corr_sets, index)
    p2._dp = DeviceProblem(len(s.ids), cl, frames, pi, pj, off)
    st2 = p2.solve(W, C, 3)
    assert [r.energy_after for r in st1.iterations] == [r.energy_after for r in st2.iterations]
    for f in s.ids:
        assert np.array_equal(p1.poses[f].rotation, p2.poses[f].rotation)
        assert np.array_equal(p1.poses[f].translation, p2.poses[f].translation)
    slots = runtime(0).slots_for(cl)
    with pytest.raises(Exception, match="already attached"):
        p1._dp.attach_frames(cl, slots)
    p1.close()
    p2.close()
