"""Device side of the column-panel split on ONE GPU: running each rank's panel
as its own gemm (no collective) must give bitwise the same C as the unsharded
call, in FAST and EXACT numerics, for every domain case -- the property that
makes the multi-GPU split reduction-free.  The collective itself is covered
by tests/test_sharded_gloo.py."""
import pytest

import paper_1901_06015_b200 as M
from paper_1901_06015_b200.sharded import gemm_sharded
from tests.helpers import Problem, SCALARS, config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("label", ["dddd", "sssd", "zzzd", "cccs", "cdds", "szzs", "zczd", "sddd", "dzsd", "zdzs"])
@pytest.mark.parametrize("numerics", ["fast", "exact"])
def test_panels_bitwise_equal_unsharded(label, numerics):
    import torch
    cfg = config({"gpu.numerics": numerics})
    for kind in ("col", "row"):
        p = Problem(label, 300, 517, 129, c_kind=kind)
        dA, dB, dC = p.device()
        full = p.C.to_device()
        va, vb, vc = p.views(A=dA, B=dB, C=dC)
        _, _, vf = p.views(A=dA, B=dB, C=full)
        M.gemm(SCALARS["cfg2_alpha_real"], va, vb, SCALARS["cfg2_beta"], vf, cfg)
        for world in (2, 3, 8):
            dC.t.copy_(torch.from_numpy(p.C.buf).cuda())
            for r in range(world):
                gemm_sharded(SCALARS["cfg2_alpha_real"], va, vb, SCALARS["cfg2_beta"], vc, cfg, world=world, rank=r)
            torch.cuda.synchronize()
            assert torch.equal(dC.t, full.t), (label, numerics, kind, world)
