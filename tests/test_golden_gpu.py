"""The device path against the committed golden fixtures: the reference
engine's own outputs (SHA-256 of C bytes, pack bytes) and the reference
tests' known answers, through the C ABI."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from tests.golden.make_golden import pack_input, run_gemm
from tests.golden_util import FMT, SIDE, load, packed_element, sha
from tests.helpers import SCALARS, config
from tests.test_golden import KATS, gemm_kat

pytestmark = pytest.mark.gpu
VECS = load("reference_vectors.json")


def device_gemm(numerics):
    def fn(alpha, a, b, beta, c, cfg):
        # operands are host views: gemm() stages them through HBM
        cfg.set("gpu.numerics", numerics)
        return M.gemm(alpha, a, b, beta, c, cfg)
    return fn


def test_exact_matches_reference_vectors():
    for rec in VECS["gemm"]:
        digest, flops = run_gemm(rec, device_gemm("exact"))
        assert digest == rec["sha256"], rec
        assert flops == rec["flops"]


def test_pack_matches_reference_vectors():
    import torch
    for rec in VECS["pack"]:
        d = pack_input(rec).to_device()
        v = d.view(conj=bool(rec["src_conj"]))
        out = torch.zeros(rec["bytes"], dtype=torch.uint8, device="cuda")
        M.pack_block_device(out.data_ptr(), v, rec["side"], rec["fmt"], rec["conj"], SCALARS[rec["scale"]],
                            rec["target"], rec["reg_block"])
        torch.cuda.synchronize()
        assert sha(out.cpu().numpy()) == rec["sha256"], rec


@pytest.mark.parametrize("kat", KATS["pack"], ids=lambda k: k["ref"])
def test_device_pack_kats(kat):
    import torch
    from tests.golden_util import matrix_from
    src = matrix_from(kat["dtype"], kat["m"], kat["n"], kat["values"]).to_device()
    v = src.view(conj=bool(kat["view_conj"]))
    tgt = M.dtype_from_letter(kat["target"])
    n = M.packed_bytes(v, SIDE[kat["side"]], FMT[kat["fmt"]], tgt, kat["reg_block"])
    out = torch.zeros(n, dtype=torch.uint8, device="cuda")
    M.pack_block_device(out.data_ptr(), v, SIDE[kat["side"]], FMT[kat["fmt"]], kat["conj"], SCALARS["one"], tgt,
                        kat["reg_block"])
    torch.cuda.synchronize()
    buf = out.cpu().numpy()
    for i, j, want in kat["expect"]:
        assert packed_element(buf, kat, i, j).real == want


@pytest.mark.parametrize("numerics", ["fast", "exact"])
@pytest.mark.parametrize("kat", KATS["gemm"], ids=lambda k: k["ref"])
def test_device_gemm_kats(kat, numerics):
    def run(al, A, B, be, C, comp):
        M.gemm(al, A.view(), B.view(), be, C.view(comp=comp), config({"gpu.numerics": numerics}))
        return C
    gemm_kat(kat, run)
