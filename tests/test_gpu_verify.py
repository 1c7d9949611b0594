"""dense_verify on the GPU (filters.dense_verify, reference filters.py:216-277).

Parity: bit-exact counts, pass flags and mean errors against the reference's
golden outputs (tests/golden/verify.npz, made by the unmodified reference) and
the CPU oracle; plus the reference's own TestDenseVerify cases
(test_filters.py:190-285) re-run through the drop-in.
"""

import copy

import numpy as np
import pytest

from golden_io import GOLDEN

pytestmark = pytest.mark.gpu

K = None


def _mods():
    from paper_1604_01093_b200 import filters as F
    from paper_1604_01093_b200 import cache as CA
    from paper_1604_01093_b200 import se3
    return F, CA, se3


def flat_cache(depth=2.0, intensity=0.4, index=0):
    """test_filters.py:52-58 with the scene generator's build_cache."""
    from scenes import host_cache as HC
    F, CA, se3 = _mods()
    k = se3.Intrinsics(525.0, 525.0, 319.5, 239.5, 640, 480)
    color = np.full((480, 640, 3), 100, dtype=np.uint8)
    frame = CA.RgbdFrame(index=index, color=color, depth=np.full((480, 640), depth, np.float32))
    c = HC.build_cache(frame, k)
    c.intensity_low[:] = intensity
    c.grad_low[:] = 0.0
    return c


def _oracle(ci, cj, T, cfg):
    from oracle import scanfuse_oracle as O
    return O.dense_verify(ci, cj, (np.asarray(T.rotation), np.asarray(T.translation)),
                          cfg.verify_depth_max, cfg.verify_normal_min, cfg.verify_color_max,
                          cfg.verify_error_max, cfg.verify_min_valid_fraction)


def _same(res, ref):
    assert res.passed == ref[0]
    assert (res.valid_count_ij, res.valid_count_ji) == (ref[3], ref[4])
    assert res.mean_error_ij == ref[1] and res.mean_error_ji == ref[2]


def test_golden_pairs_bit_exact():
    F, CA, se3 = _mods()
    from scenes import synth
    sc = synth.make("cfg3")
    g = np.load(GOLDEN / "verify.npz")
    pairs = []
    for k, (a, b) in enumerate(g["pairs"]):
        R = g["R"][k]
        R = np.asfortranarray(R) if g["f_order"][k] else np.ascontiguousarray(R)
        pairs.append((sc.caches[int(a)], sc.caches[int(b)], se3.RigidTransform(R, g["t"][k].copy())))
    res = F.dense_verify_many(pairs, F.FilterConfig())
    assert len(res) == len(pairs)
    for k, r in enumerate(res):
        assert r.passed == bool(g["passed"][k]), k
        assert r.valid_count_ij == int(g["count_ij"][k]), k
        assert r.valid_count_ji == int(g["count_ji"][k]), k
        assert r.mean_error_ij == g["err_ij"][k], k
        assert r.mean_error_ji == g["err_ji"][k], k
    # the single-pair entry point agrees with the batched one
    one = F.dense_verify(*pairs[5], F.FilterConfig())
    assert one == res[5]


def test_error_max_override_and_oracle():
    F, CA, se3 = _mods()
    from scenes import synth
    sc = synth.make("cfg3")
    T = sc.truth[20].inverse().compose(sc.truth[17])
    cfg = F.FilterConfig()
    for em in (None, 0.05, 1e-9):
        r = F.dense_verify(sc.caches[17], sc.caches[20], T, cfg, error_max=em)
        ref = _oracle(sc.caches[17], sc.caches[20], T, cfg if em is None else
                      F.FilterConfig(verify_error_max=em))
        _same(r, ref)


class TestReferenceDenseVerify:
    """test_filters.py:190-285 through the drop-in."""

    def test_self_pair_identity(self):
        F, CA, se3 = _mods()
        cache = flat_cache()
        r = F.dense_verify(cache, cache, se3.RigidTransform.identity(), F.FilterConfig())
        eligible = int(np.count_nonzero(cache.valid_depth & cache.valid_normal))
        assert r.passed
        assert r.mean_error_ij == 0.0 and r.mean_error_ji == 0.0
        assert r.valid_count_ij == eligible and r.valid_count_ji == eligible

    def test_large_axial_offset_fails(self):
        F, CA, se3 = _mods()
        cache = flat_cache()
        moved = se3.RigidTransform(np.eye(3), np.array([0.0, 0.0, 0.3]))
        assert not F.dense_verify(cache, cache, moved, F.FilterConfig()).passed

    def test_depth_gate_both_sides(self):
        F, CA, se3 = _mods()
        base = flat_cache()
        for delta, full in ((0.149, True), (0.151, False)):
            other = copy.deepcopy(base)
            other.points_low[..., 2] += delta
            other.depth_low += delta
            r = F.dense_verify(base, other, se3.RigidTransform.identity(), F.FilterConfig())
            n = int(np.count_nonzero(base.valid_depth & base.valid_normal))
            assert r.valid_count_ij == (n if full else 0)
            _same(r, _oracle(base, other, se3.RigidTransform.identity(), F.FilterConfig()))

    def test_normal_gate_both_sides(self):
        F, CA, se3 = _mods()
        base = flat_cache()
        for cosine, full in ((0.91, True), (0.89, False)):
            other = copy.deepcopy(base)
            R = se3.so3_exp(np.array([np.arccos(cosine), 0.0, 0.0]))
            other.normals_low = (other.normals_low.reshape(-1, 3) @ R.T).reshape(
                other.normals_low.shape).astype(np.float32)
            r = F.dense_verify(base, other, se3.RigidTransform.identity(), F.FilterConfig())
            assert (r.valid_count_ij > 0) == full
            _same(r, _oracle(base, other, se3.RigidTransform.identity(), F.FilterConfig()))

    def test_color_gate_both_sides(self):
        F, CA, se3 = _mods()
        base = flat_cache(intensity=0.4)
        for diff, full in ((0.09, True), (0.11, False)):
            other = copy.deepcopy(base)
            other.intensity_low[:] = 0.4 + diff
            r = F.dense_verify(base, other, se3.RigidTransform.identity(), F.FilterConfig())
            assert (r.valid_count_ij > 0) == full
            _same(r, _oracle(base, other, se3.RigidTransform.identity(), F.FilterConfig()))

    def test_mean_error_gate_both_sides(self):
        F, CA, se3 = _mods()
        base = flat_cache()
        for delta, ok in ((0.074, True), (0.076, False)):
            other = copy.deepcopy(base)
            other.points_low[..., 0] += delta
            r = F.dense_verify(base, other, se3.RigidTransform.identity(), F.FilterConfig())
            assert r.passed == ok
            assert r.mean_error_ij == pytest.approx(delta, rel=1e-5)
            _same(r, _oracle(base, other, se3.RigidTransform.identity(), F.FilterConfig()))

    def test_min_valid_count_boundary(self):
        F, CA, se3 = _mods()
        for count, ok in ((96, True), (95, False)):
            cache = flat_cache()
            keep = np.zeros_like(cache.valid_depth)
            ys, xs = np.nonzero(cache.valid_depth & cache.valid_normal)
            keep[ys[:count], xs[:count]] = True
            cache.valid_depth &= keep
            cache.valid_normal &= keep
            r = F.dense_verify(cache, cache, se3.RigidTransform.identity(), F.FilterConfig())
            assert r.valid_count_ij == count
            assert r.passed == ok

    def test_half_overlap_plane_views(self):
        F, CA, se3 = _mods()
        cache = flat_cache(depth=2.0)
        width = 80 * 2.0 / cache.intrinsics_low.fx
        rel = se3.RigidTransform(np.eye(3), np.array([-width / 2, 0.0, 0.0]))
        r = F.dense_verify(cache, cache, rel, F.FilterConfig())
        n = int(np.count_nonzero(cache.valid_depth & cache.valid_normal))
        assert r.passed
        assert 0.35 * n < r.valid_count_ij < 0.65 * n
        assert r.mean_error_ij < 1e-4
        _same(r, _oracle(cache, cache, rel, F.FilterConfig()))

    def test_two_sided_symmetry(self):
        F, CA, se3 = _mods()
        cache = flat_cache(depth=2.0)
        shift = se3.RigidTransform(np.eye(3), np.array([-0.4, 0.05, 0.0]))
        fwd = F.dense_verify(cache, cache, shift, F.FilterConfig())
        bwd = F.dense_verify(cache, cache, shift.inverse(), F.FilterConfig())
        assert fwd.passed == bwd.passed
        assert fwd.valid_count_ij == bwd.valid_count_ji


def test_no_eligible_pixels_and_single_pixel():
    """filters.py:219-221 (no eligible pixel -> (0.0, 0)) and the m == 1
    rounding path (NumPy's gemv order for a single eligible pixel)."""
    F, CA, se3 = _mods()
    empty = flat_cache()
    empty.valid_depth[:] = False
    full = flat_cache()
    T = se3.RigidTransform(se3.so3_exp(np.array([0.01, -0.02, 0.005])), np.array([0.01, 0.0, 0.02]))
    r = F.dense_verify(empty, full, T, F.FilterConfig())
    assert (r.valid_count_ij, r.mean_error_ij) == (0, 0.0) and not r.passed
    one = flat_cache()
    keep = np.zeros_like(one.valid_depth)
    ys, xs = np.nonzero(one.valid_depth & one.valid_normal)
    keep[ys[40], xs[40]] = True
    one.valid_depth &= keep
    one.valid_normal &= keep
    for rot in (np.ascontiguousarray(T.rotation), np.asfortranarray(T.rotation)):
        X = se3.RigidTransform(rot, T.translation.copy())
        _same(F.dense_verify(one, full, X, F.FilterConfig()),
              _oracle(one, full, X, F.FilterConfig()))
