"""Hashed TSDF on the GPU (paper_1604_01093_b200.tsdf, reference tsdf.py:55-267).

Parity: after every integrate / de-integrate of the golden scenarios the
device volume's blocks (coordinates, float32 accumulators, dict insertion
order) hash to the digests the unmodified reference produced
(tests/golden/tsdf_digests.json), and de-integration mismatches raise the
same error at the same block.  Plus the read API against the CPU oracle.
"""

import json
import re
import sys

import numpy as np
import pytest

from golden_io import GOLDEN

sys.path.insert(0, str(GOLDEN))
from make_tsdf_golden import SCENARIOS, tsdf_inputs, volume_digest  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(name, steps_out=None):
    from paper_1604_01093_b200 import se3
    from paper_1604_01093_b200 import tsdf as T
    from paper_1604_01093_b200.cache import RgbdFrame
    frames, K, truth, noisy = tsdf_inputs()
    k = se3.Intrinsics(*K)
    vs, trunc, dw, steps = SCENARIOS[name]
    v = T.TsdfVolume(vs, trunc, dw)
    recs = []
    for fi, sign, nz in steps:
        col, dep = frames[fi]
        R, t = (noisy if nz else truth)[fi]
        err = None
        try:
            (v.integrate if sign > 0 else v.deintegrate)(RgbdFrame(fi, col, dep), k,
                                                         se3.RigidTransform(R, t))
        except T.DeintegrationMismatchError as e:
            err = str(e)
        blocks = v.blocks
        d = volume_digest(list(blocks), {c: (b.weight, b.wdist, b.wcolor) for c, b in blocks.items()})
        d["error"] = err
        recs.append(d)
    return v, recs


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_tsdf_matches_reference_digests(name):
    g = json.loads((GOLDEN / "tsdf_digests.json").read_text())[name]
    _, recs = _run(name)
    for step, (got, exp) in enumerate(zip(recs, g)):
        for key in ("blocks", "occupied", "data", "order"):
            assert got[key] == exp[key], (name, step, key, got[key], exp[key])
        assert (got["error"] is None) == (exp["error"] is None), (step, got["error"], exp["error"])
        if exp["error"] is not None:  # same block, same wording (modulo numpy's int repr)
            nums = lambda m: [int(x) for x in re.findall(r"-?\d+", m.replace("np.int64", ""))]
            assert nums(got["error"]) == nums(exp["error"]), (got["error"], exp["error"])
            assert got["error"].split("(")[0] == exp["error"].split("(")[0]

def test_tsdf_read_api_save_load_and_oracle(tmp_path):
    from oracle import scanfuse_oracle as O
    from paper_1604_01093_b200 import se3
    from paper_1604_01093_b200 import tsdf as T
    v, _ = _run("vs20")
    frames, K, truth, noisy = tsdf_inputs()
    o = O.TsdfOracle(0.02)
    for fi, sign, nz in SCENARIOS["vs20"][3]:
        o.apply_frame(frames[fi][0], frames[fi][1], se3.Intrinsics(*K), truth[fi], sign)
    blocks = v.blocks
    assert list(blocks) == list(o.blocks)
    assert v.sorted_coords() == sorted(o.blocks)
    assert v.occupied_voxel_count() == sum(int(np.count_nonzero(b[0])) for b in o.blocks.values())
    rng = np.random.default_rng(5)
    cs = list(o.blocks)
    for _ in range(50):
        c = cs[rng.integers(len(cs))]
        p = (np.array(c) + rng.random(3)) * v.block_extent
        d, w = v.voxel_state(p)
        blk = o.blocks[c]
        loc = np.floor(p / 0.02).astype(int) - np.array(c) * 8
        idx = loc[0] * 64 + loc[1] * 8 + loc[2]
        if blk[0][idx] > 0:
            assert w == float(blk[0][idx]) and d == float(blk[1][idx] / blk[0][idx])
        else:
            assert (d, w) == (None, 0.0)
    assert v.block((10 ** 6, 0, 0)) is None
    b0 = v.block(cs[0])
    assert np.array_equal(b0.weight, o.blocks[cs[0]][0])
    path = tmp_path / "vol.npz"
    T.save_volume(path, v)
    v2 = T.load_volume(path)
    assert T.volumes_equal(v, v2, 0.0)
    assert v2.sorted_coords() == v.sorted_coords()
    n = len(v2)
    e = v2.allocate((10 ** 5, 3, -7))
    assert len(v2) == n + 1 and not e.weight.any()
    assert list(v2.blocks)[-1] == (10 ** 5, 3, -7)


def test_tsdf_blocks_view_writes_through_and_is_read_only():
    """`blocks` is a live view (single-block fetches, write-through
    assignment, cache invalidated by integrate) and handed-out arrays raise on
    writes instead of silently losing them."""
    from paper_1604_01093_b200 import tsdf as T
    v, _ = _run("vs20")
    view = v.blocks
    coords = list(view)
    snap = v.snapshot()
    assert coords == list(snap)
    c = coords[len(coords) // 2]
    b = view[c]
    assert np.array_equal(b.weight, snap[c].weight) and np.array_equal(b.wcolor, snap[c].wcolor)
    assert view[c] is b  # cached until the volume changes
    with pytest.raises(ValueError):
        b.weight[0] = 1.0
    new = T.VoxelBlock(np.full(T.BLOCK_VOXELS, 2.0, np.float32), np.full(T.BLOCK_VOXELS, 0.5, np.float32),
                       np.ones((T.BLOCK_VOXELS, 3), np.float32))
    view[c] = new
    got = v.blocks[c]
    assert got is not b and np.array_equal(got.weight, new.weight) and np.array_equal(got.wdist, new.wdist)
    assert list(v.blocks) == coords  # overwrite keeps the insertion order
    view[(7, 7, 7777)] = new
    assert list(v.blocks)[-1] == (7, 7, 7777) and (7, 7, 7777) in v.blocks
    assert v.block((1, 2, 10 ** 6)) is None and (1, 2, 10 ** 6) not in v.blocks
    with pytest.raises(TypeError):
        del view[c]
