"""Maximum sizes: views with more than 2**31 elements (and 2**32 bytes).

The reference indexes with 64-bit integers throughout (`MatrixView` strides
and offsets are int64_t, `include/mdgemm/types.hpp`); these cases check that
no 32-bit product survives in the B200 path -- C tiles far past element 2**31
(real and 1m complex images, both warp-specialised kernels), and an inner
dimension long enough that the packed panels pass 2**31 elements.  Checked
like the BASELINE-scale tests: sampled rows/columns (edges included) against
the oracle with the full inner dimension."""
import pytest

import paper_1901_06015_b200 as M
from tests.test_baseline_scale_gpu import run_config

pytestmark = pytest.mark.gpu


def _free():
    import torch
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("label,m,n,k", [
    ("ssss", 49152, 49152, 32),   # C: 2.4e9 floats (9.7 GB), FFMA WS kernel
    ("sddd", 49152, 49152, 32),   # C: 2.4e9 floats, DMMA WS kernel
    ("zzzd", 34816, 34816, 32),   # C: 1.2e9 complex = 2.4e9 doubles in the 1m real image
])
def test_c_past_2_31_elements(label, m, n, k):
    assert m * n * (2 if label[0] in "cz" else 1) > 2**31
    one, beta = M.Scalar.real_value(1.0), M.Scalar.real_value(0.5)
    run_config(label, m, n, k, one, beta, "fast", seed=7, nsamp=10)
    _free()


def test_exact_c_past_2_31_elements():
    # the EXACT replay kernel (gemm_exact.cu): bitwise the reference on sampled blocks
    one, beta = M.Scalar.real_value(1.0), M.Scalar.complex_value(0.5, 0.25)
    run_config("sdds", 49152, 49152, 8, one, beta, "exact", seed=5, nsamp=8, exact_bitwise=True)
    _free()


def test_inner_dimension_past_2_31_packed_elements():
    # A is 192 x 12e6 floats: the left pack's panel offsets pass 2**31 elements
    m = n = 192
    k = 12_000_000
    assert m * k > 2**31
    run_config("ssss", m, n, k, M.Scalar.real_value(1.0), M.Scalar.real_value(0.0), "fast", seed=8, nsamp=6)
    _free()


def test_dual_batch_past_2_31_elements(monkeypatch):
    """A mixed-precision batch on the dual-pipe kernel whose FP64 and FP32 calls each
    have a C past 2**31 elements: bitwise equal to calling gemm() on each."""
    import torch
    from tests.test_baseline_scale_gpu import DevMat
    monkeypatch.setenv("MDGEMM_DUAL", "1")
    cfg = M.Config.defaults()
    m = n = 49152
    k = 32
    one, beta = M.Scalar.real_value(1.0), M.Scalar.real_value(0.5)
    mats = {}
    for label in ("sddd", "ssss"):
        dc, da, db = (M.dtype_from_letter(ch) for ch in label[:3])
        root = M.Rng(9).split(label)
        mats[label] = (DevMat(da, m, k, root.split("a").state), DevMat(db, k, n, root.split("b").state),
                       DevMat(dc, m, n, root.split("c").state), M.SINGLE if label[3] == "s" else M.DOUBLE)
    want = {}
    for label, (A, B, C, comp) in mats.items():
        c = C.copy()
        M.gemm(one, A.view(), B.view(), beta, c.view(comp), cfg)
        want[label] = c
    M.profile_begin()
    M.gemm_batch([(one, A.view(), B.view(), beta, C.view(comp)) for A, B, C, comp in mats.values()], cfg)
    ks = M.profile_end()
    torch.cuda.synchronize()
    assert ks["dual_d"]["launches"] > 0 and ks["dual_f"]["work"] > 0, ks  # one launch, both groups
    for label, (A, B, C, comp) in mats.items():
        assert torch.equal(C.t, want[label].t), label
    del mats, want
    _free()
