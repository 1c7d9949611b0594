"""The persistent PCG with each block row summed by SPLIT = 1, 2, 4 or 8 warps
(`k_pcg_reg<.., SPLIT>`; the launcher picks the widest split whose grid fits
the SMs, SFB_PCG_SPLIT forces one).  Every split must reproduce the
reference's PCG on the golden linearisation (iteration count, residual, x) -
the splits differ only in the order the row products are added."""
import os

import numpy as np
import pytest

from golden_io import GoldenScene
from paper_1604_01093_b200 import solver as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["cfg2", "cfg3"])
def system(request):
    scene = GoldenScene(request.param)
    g = scene.g
    p = S.AlignmentProblem(scene.ids, scene.init, scene.corr_sets, scene.caches)
    p.dense_edges = [tuple(e) for e in g["edges"].tolist()]
    w, cfg = scene.weights_obj(S), scene.config_obj(S)
    eqs, _, _, _ = p.normal_equations(w, 1.0, cfg)
    return g, eqs, cfg


@pytest.mark.parametrize("split", [1, 2, 4, 8])
def test_pcg_split_matches_reference(system, split):
    g, eqs, cfg = system
    old = os.environ.get("SFB_PCG_SPLIT")
    os.environ["SFB_PCG_SPLIT"] = str(split)
    try:
        x, info = S.pcg_solve(eqs, cfg.pcg_max_iterations, cfg.pcg_tolerance, cfg.pcg_restart_interval)
    finally:
        if old is None:
            del os.environ["SFB_PCG_SPLIT"]
        else:
            os.environ["SFB_PCG_SPLIT"] = old
    assert info.iterations == int(g["pcg_info"][0])
    assert info.relative_residual == pytest.approx(g["pcg_info"][1], rel=1e-6)
    np.testing.assert_allclose(x, g["pcg_x"], rtol=0, atol=1e-7 * np.abs(g["pcg_x"]).max())
