"""FAST numerics honour ctemp.enable = off.

Without C_temp the reference rounds each KC block's partial sum into C
(Temp path: one accumulate_element per block, beta on the first and 1 after,
gemm_core.cpp:125-127, kernels.cpp:97-132; 1m with a complex beta: the first
block through the temp tile, the rest continued in the computation precision,
kernels.cpp:141-150).  Where C is stored at another precision than the
computation's, FAST runs one kernel pass per KC block (driver.cpp:
fast_block_mode), so each block's sum meets C's storage rounding exactly where
the reference's does; where the precisions agree the block boundaries only
reorder the sum in the computation precision and FAST keeps one pass.  Checked against the oracle run with the same Config
(per-element criterion, north-star Frobenius bound) and against EXACT: where
C's storage precision is narrower than the computation precision (the
per-block sums are rounded to storage), every element is within one storage
ulp of the bitwise-reference EXACT result."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import Problem, SCALARS, config, frob_bound, label_dtypes, rel_frobenius, ulp_distance

pytestmark = pytest.mark.gpu

LABELS = ["zzzd", "cccs", "zczd", "czzs", "zdzd", "dzzd", "sddd", "cdds", "ssds", "sdds", "czzd", "cddd"]


def run(p, alpha, beta, kv):
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    flops = M.gemm(alpha, da, db, beta, dc, config(kv))
    out = p.C.clone()
    out.buf[:] = dC.bytes()
    return out, flops


@pytest.mark.parametrize("label", LABELS)
@pytest.mark.parametrize("shape_kc", [((12, 8, 40), 16), ((70, 50, 300), 64), ((130, 129, 1000), 128)])
def test_fast_ctemp_off_rounds_per_kc_block(label, shape_kc):
    (m, n, k), kc = shape_kc
    dc, _, _, comp = label_dtypes(label)
    kv = {"gemm.kc": str(kc), "ctemp.enable": "off"}
    for be in ("cfg2_beta", "p3", "one", "zero"):
        alpha = SCALARS["cfg2_alpha_real"]
        p = Problem(label, m, n, k, variant=f"off{kc}")
        fast, f_fast = run(p, alpha, SCALARS[be], {**kv, "gpu.numerics": "fast"})
        exact, f_exact = run(p, alpha, SCALARS[be], {**kv, "gpu.numerics": "exact"})
        want = p.C.clone()
        va, vb, vw = p.views(C=want)
        f_ref = O.orc_gemm(alpha, va, vb, SCALARS[be], vw, config(kv))
        assert f_fast == f_exact == f_ref
        assert exact.buf.tobytes() == want.buf.tobytes()  # EXACT is the reference, bit for bit
        _, _, vc = p.views()
        _, _, vf = p.views(C=fast)
        assert O.orc_violation(alpha, va, vb, SCALARS[be], vc, vf, p.comp) <= 1.0
        assert rel_frobenius(fast.values(), want.values()) <= frob_bound(label, k)
        if M.precision_of(dc) == M.SINGLE and comp == M.DOUBLE:  # storage narrower than the sums
            d = ulp_distance(fast.values(), want.values())
            assert int(d.max()) <= 1, (label, be, int(d.max()))


def test_fast_ctemp_off_differs_from_ctemp_on_where_the_reference_does():
    # sddd: C single, computation double.  With C_temp the fp64 sum is rounded to float once;
    # without it once per KC block.  FAST must follow the Config, like the reference.
    p = Problem("sddd", 64, 64, 2048, variant="onoff")
    alpha, beta = SCALARS["one"], SCALARS["one"]
    res = {}
    for mode in ("on", "off"):
        kv = {"gemm.kc": "64", "ctemp.enable": mode}
        fast, _ = run(p, alpha, beta, {**kv, "gpu.numerics": "fast"})
        want = p.C.clone()
        va, vb, vw = p.views(C=want)
        O.orc_gemm(alpha, va, vb, beta, vw, config(kv))
        res[mode] = (fast, want)
    assert res["on"][1].buf.tobytes() != res["off"][1].buf.tobytes()  # the reference differs
    for mode in ("on", "off"):
        fast, want = res[mode]
        assert int(ulp_distance(fast.values(), want.values()).max()) <= 1, mode
    # each FAST result is far closer to its own mode's reference than to the other mode's
    for mode, other in (("on", "off"), ("off", "on")):
        mine = ulp_distance(res[mode][0].values(), res[mode][1].values()).sum()
        cross = ulp_distance(res[mode][0].values(), res[other][1].values()).sum()
        assert mine < cross, (mode, mine, cross)
