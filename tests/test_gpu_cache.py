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
    from scenes import host_cache as HC
    from paper_1604_01093_b200 import se3
    g = json.loads((GOLDEN / "cache_digests.json").read_text())
    checked = 0
    for (shape, (lw, lh), kk), items in _groups().items():
        k = se3.Intrinsics(*kk)
        frames = [CA.RgbdFrame(i, col, dep) for i, (_, col, dep) in enumerate(items)]
        dev = CA.build_cache_device(frames, k, lw, lh)
        for (name, col, dep), c in zip(items, dev):
            host = HC.build_cache(CA.RgbdFrame(0, col, dep), k, lw, lh)
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
    from scenes import host_cache as HC
    from paper_1604_01093_b200 import se3
    from scenes import synth
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
    from scenes import host_cache as HC
    from paper_1604_01093_b200 import filters as F
    from paper_1604_01093_b200 import se3
    from scenes import synth
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


class TestReferenceBuildCache:
    """test_frames.py:17-80 through build_cache_device (and equal to the host
    build_cache on each input)."""

    @staticmethod
    def _k():
        from paper_1604_01093_b200 import se3
        return se3.Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)

    @staticmethod
    def _frame(depth_value=2.0, index=0, color=None):
        from paper_1604_01093_b200.cache import RgbdFrame
        depth = np.full((480, 640), depth_value, dtype=np.float32)
        if color is None:
            rng = np.random.default_rng(index + 1)
            color = rng.integers(0, 255, size=(480, 640, 3), dtype=np.uint8)
        return RgbdFrame(index=index, color=color, depth=depth)

    def _dev(self, frame):
        from paper_1604_01093_b200 import cache as CA
        from scenes import host_cache as HC
        c = CA.build_cache_device([frame], self._k())[0]
        h = HC.build_cache(frame, self._k())
        for p in PLANES:
            a, b = np.asarray(getattr(c, p)), np.asarray(getattr(h, p))
            assert a.dtype == b.dtype and np.array_equal(a, b), p
        return c

    def test_planar_frame_normals(self):
        cache = self._dev(self._frame(depth_value=2.0))
        ok = cache.valid_normal
        assert np.count_nonzero(ok) > 0.9 * ok.size
        assert np.allclose(cache.normals_low[ok], [0.0, 0.0, -1.0], atol=1e-3)

    def test_all_invalid_depth(self):
        frame = self._frame()
        frame.depth[:] = 0.0
        cache = self._dev(frame)
        assert np.count_nonzero(cache.valid_depth) == 0
        assert np.count_nonzero(cache.valid_normal) == 0

    def test_intensity_ramp_gradient(self):
        xs = np.arange(640, dtype=np.float32) / 640.0
        gray = np.tile((xs * 255).astype(np.uint8), (480, 1))
        cache = self._dev(self._frame(color=np.repeat(gray[..., None], 3, axis=2)))
        interior = cache.grad_low[5:-5, 5:-5]
        expected = 1.0 / 80.0
        assert np.all(np.abs(interior[..., 0] - expected) < 0.05 * expected)
        assert np.all(np.abs(interior[..., 1]) < 1e-4)

    def test_points_match_unprojection(self):
        cache = self._dev(self._frame())
        ys, xs = np.nonzero(cache.valid_depth)
        pix = np.stack([xs, ys], axis=-1).astype(np.float64)
        expected = cache.intrinsics_low.unproject(pix, cache.depth_low[ys, xs])
        assert np.allclose(cache.points_low[ys, xs], expected.astype(np.float32))

    def test_points_reproject_to_pixel_centers(self):
        frame = self._frame()
        rng = np.random.default_rng(0)
        frame.depth += rng.uniform(-0.2, 0.2, size=frame.depth.shape).astype(np.float32)
        cache = self._dev(frame)
        ys, xs = np.nonzero(cache.valid_depth)
        pix, in_front = cache.intrinsics_low.project_many(cache.points_low[ys, xs].astype(np.float64))
        assert np.all(in_front)
        assert np.all(np.abs(pix[:, 0] - xs) < 0.5) and np.all(np.abs(pix[:, 1] - ys) < 0.5)

    def test_deterministic(self):
        frame = self._frame(index=3)
        a, b = self._dev(frame), self._dev(frame)
        for p in PLANES:
            assert np.array_equal(getattr(a, p), getattr(b, p))

    def test_median_ignores_invalid_samples(self):
        frame = self._frame(depth_value=2.0)
        frame.depth[0:8, 0:8] = 0.0
        frame.depth[0, 0] = 2.0
        assert self._dev(frame).depth_low[0, 0] == np.float32(2.0)
