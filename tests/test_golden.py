"""The oracle against the committed golden fixtures: the reference tests'
known answers (tests/golden/kats.json) and the vectors the reference engine
produced (tests/golden/reference_vectors.json, tests/golden/make_golden.py).
CPU only; the GPU counterpart is test_golden_gpu.py."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.golden.make_golden import GEMM_SPECS, PACK_SPECS, pack_input, run_gemm
from tests.golden_util import FMT, SIDE, load, matrix_from, packed_element, sha
from tests.helpers import SCALARS

KATS = load("kats.json")
VECS = load("reference_vectors.json")


def test_fixture_specs_match_generator():
    assert len(VECS["gemm"]) == len(GEMM_SPECS) and len(VECS["pack"]) == len(PACK_SPECS)


@pytest.mark.parametrize("kat", KATS["pack"], ids=lambda k: k["ref"])
def test_oracle_pack_kats(kat):
    src = matrix_from(kat["dtype"], kat["m"], kat["n"], kat["values"])
    v = src.view(conj=bool(kat["view_conj"]))
    tgt = M.dtype_from_letter(kat["target"])
    n = O.orc_packed_bytes(v, SIDE[kat["side"]], FMT[kat["fmt"]], tgt, kat["reg_block"])
    buf = np.zeros(n, np.uint8)
    O.orc_pack(v, SIDE[kat["side"]], FMT[kat["fmt"]], kat["conj"], SCALARS["one"], tgt, kat["reg_block"], 0,
               buf.ctypes.data)
    for i, j, want in kat["expect"]:
        assert packed_element(buf, kat, i, j).real == want


def gemm_kat(kat, runner):
    lab = kat["label"]
    comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
    A = matrix_from(lab[1], kat["m"], kat["k"], kat["A"])
    B = matrix_from(lab[2], kat["k"], kat["n"], kat["B"])
    C = matrix_from(lab[0], kat["m"], kat["n"], kat["C"])
    al = M.Scalar.complex_value(*kat["alpha"]) if kat["alpha"][1] else M.Scalar.real_value(kat["alpha"][0])
    be = M.Scalar.complex_value(*kat["beta"]) if kat["beta"][1] else M.Scalar.real_value(kat["beta"][0])
    out = runner(al, A, B, be, C, comp)
    vals = out.values().reshape(-1, order="F")
    if "expect_f32" in kat:
        want = [complex(np.float32(r), np.float32(i)) for r, i in kat["expect_f32"]]
    else:
        want = [complex(r, i) for r, i in kat["expect"]]
    assert [complex(v) for v in vals] == want, kat["ref"]


@pytest.mark.parametrize("kat", KATS["gemm"], ids=lambda k: k["ref"])
def test_oracle_gemm_kats(kat):
    def run(al, A, B, be, C, comp):
        O.orc_gemm(al, A.view(), B.view(), be, C.view(comp=comp))
        return C
    gemm_kat(kat, run)


def test_oracle_reproduces_reference_vectors():
    for rec in VECS["gemm"]:
        digest, flops = run_gemm(rec, O.orc_gemm)
        assert digest == rec["sha256"], rec
        assert flops == rec["flops"]
    for rec in VECS["pack"]:
        src = pack_input(rec)
        v = src.view(conj=bool(rec["src_conj"]))
        buf = np.zeros(rec["bytes"], np.uint8)
        O.orc_pack(v, rec["side"], rec["fmt"], rec["conj"], SCALARS[rec["scale"]], rec["target"], rec["reg_block"], 0,
                   buf.ctypes.data)
        assert sha(buf) == rec["sha256"], rec
