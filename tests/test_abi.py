"""The drop-in boundary: the C-ABI library loads without a GPU and exports
every entry point include/mdgemm_b200.h declares; host-only entry points
behave like the reference (no device work is done here)."""
import ctypes
import os
import re

import pytest

import paper_1901_06015_b200 as M
from tests.helpers import SCALARS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mdgemm_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mdg_[a-z_0-9]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1901_06015_b200", "libmdgemm_b200.so"))
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(M.EXPORTED_SYMBOLS)


def test_abi_version_and_struct_sizes():
    assert M.lib.mdg_abi_version() == 2  # 2: mdg_config_t gained gpu.splitk
    assert ctypes.sizeof(M.MatrixView) == 56
    assert ctypes.sizeof(M.Scalar) == 24
    assert ctypes.sizeof(M.Config) == 88


def test_oracle_abi_mirror_matches_the_product_layout():
    # the checkers declare the structs themselves (oracle/abi.py), so that the reference
    # arm never loads the product library: same field names, offsets and sizes
    from oracle import abi as A
    for mine, theirs in ((M.MatrixView, A.MatrixView), (M.Scalar, A.Scalar), (M.Config, A.Config),
                         (M.ExecutionPlan, A.ExecutionPlan)):
        assert ctypes.sizeof(mine) == ctypes.sizeof(theirs), mine
        for (name, _), (name2, _) in zip(mine._fields_, theirs._fields_):
            assert name == name2 and getattr(mine, name).offset == getattr(theirs, name2).offset, (mine, name)
    for c in (0, 1):
        for a in (0, 1):
            for b in (0, 1):
                label = "dz"[c] + "dz"[a] + "dz"[b] + "d"
                assert A.case_id(label) == M.classify_case(bool(c), bool(a), bool(b))
    assert A.flops_of_case(7, 3, 5, 7) == M.flops_of_case(7, 3, 5, 7)
    assert A.all_labels() == [l.str() for l in M.CaseLabel.all()]
    h = A.HostMatrix(M.DT_C, 5, 3)
    assert bytes(h.view()) == bytes(M.MatrixView.make(h.buf.ctypes.data, 5, 3, 1, 5, M.DT_C))


def test_config_keys_and_errors():
    cfg = M.Config.defaults()
    assert (cfg.double_params.mr, cfg.double_params.kc, cfg.single_params.nc) == (4, 128, 1024)
    cfg.set("gemm.kc.double", 64).set("ukr.preference", "row").set("ctemp.enable", "off").set("gpu.numerics", "exact")
    assert cfg.double_params.kc == 64 and cfg.single_params.kc == 256
    assert (cfg.preference, cfg.ctemp, cfg.numerics) == (M.PREF_ROW, M.CTEMP_OFF, M.EXACT)
    assert cfg.splitk == 1 and M.Config.defaults().set("gpu.splitk", "off").splitk == 0
    for key, val in (("gemm.bogus", "1"), ("ukr.preference", "diagonal"), ("gemm.kc", "x12"),
                     ("ctemp.enable", "sometimes"), ("gpu.numerics", "approx"), ("gpu.splitk", "maybe")):
        with pytest.raises(M.Error):
            M.Config.defaults().set(key, val)
    bad = M.Config.defaults().set("ukr.mr", 3)
    with pytest.raises(M.Error):
        bad.validate()


def test_config_load_file_and_env(tmp_path, monkeypatch):
    path = tmp_path / "mdgemm.conf"
    path.write_text("# comment\ngemm.threads = 4\nukr.nr.single=16\n")
    monkeypatch.setenv("MDGEMM_CTEMP_ENABLE", "on")
    monkeypatch.setenv("MDGEMM_GPU_NUMERICS", "exact")
    cfg = M.Config.load(str(path))
    assert (cfg.threads, cfg.single_params.nr, cfg.ctemp, cfg.numerics) == (4, 16, M.CTEMP_ON, M.EXACT)
    path.write_text("not a key value line\n")
    with pytest.raises(M.Error):
        M.Config.load(str(path))


def test_view_validation():
    with pytest.raises(M.Error):
        M.MatrixView.make(0x1000, 4, 4, 1, 3, M.DT_D)  # aliasing strides
    with pytest.raises(M.Error):
        M.MatrixView.make(0x1000, -1, 4, 1, 4, M.DT_D)
    with pytest.raises(M.Error):
        M.MatrixView.make(0x1000, 4, 4, 0, 4, M.DT_D)
    v = M.MatrixView.make(0x1000, 4, 5, 1, 4, M.DT_Z)
    assert (v.comp_prec, v.target_dtype) == (M.DOUBLE, M.DT_Z)


def test_case_table_and_flops():
    # acceptance.cpp:78-96
    table = {(0, 0, 0): 0, (0, 1, 0): 1, (0, 0, 1): 2, (1, 0, 0): 3, (0, 1, 1): 4, (1, 1, 0): 5, (1, 0, 1): 6, (1, 1, 1): 7}
    for (c, a, b), want in table.items():
        assert M.classify_case(c, a, b) == want
    assert [M.flops_of_case(i, 2, 3, 5) for i in range(8)] == [60, 60, 60, 60, 120, 120, 120, 240]


def test_scalar_policy():
    a, b = M.apply_scalar_policy(SCALARS["c55"], SCALARS["c34"], 0, M.SINGLE, M.DOUBLE)
    assert (a.re, a.im, a.dtype, b.re, b.im) == (0.5, 0.0, M.DT_S, 0.3, 0.0)
    a, b = M.apply_scalar_policy(SCALARS["c55"], SCALARS["c34"], 7, M.SINGLE, M.DOUBLE)
    assert a.dtype == M.DT_C and a.im == 0.5 and b.im == 0.4
    with pytest.raises(M.ScalarPolicyError):
        M.apply_scalar_policy(SCALARS["c55"], SCALARS["one"], 5, M.DOUBLE, M.DOUBLE)


def test_labels():
    labels = M.CaseLabel.all()
    assert len(labels) == 128 and labels[0].str() == "ssss" and labels[-1].str() == "zzzd"
    assert M.CaseLabel.parse("zcsd").case_id() == 5
    with pytest.raises(M.Error):
        M.CaseLabel.parse("zcs")


def test_shard_columns():
    for n, world, align in ((1000, 3, 8), (16384, 8, 128), (7, 4, 1), (5, 8, 4)):
        spans = [M.shard_columns(n, world, r, align) for r in range(world)]
        assert sum(nb for _, nb in spans) == n
        pos = 0
        for j0, nb in spans:
            assert j0 == pos or nb == 0
            pos = j0 + nb
