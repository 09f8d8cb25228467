"""The library's multi-GPU entry points on one B200:
mdg_gemm_sharded through a one-rank NCCL communicator and mdg_gemm_multi on
one device.  Panels are run one after another (no rank waits on another's
kernels on the same GPU); every assembled result must equal the unsharded
call bit for bit (both without split-K: a shard never splits, and gpu.splitk
= off keeps the unsharded call on the whole-k grid), including a long inner
dimension with few columns where the unsharded call would otherwise split,
transposed plans (row-major C, case 2bc) and host operands."""
import numpy as np
import pytest

import paper_1901_06015_b200 as M
from tests.helpers import Problem, SCALARS, config

pytestmark = pytest.mark.gpu

CASES = [("dddd", 300, 290, 129, "col"), ("zzzd", 130, 257, 70, "col"), ("cdds", 64, 80, 1100, "col"),
         ("zdzs", 90, 140, 33, "row"), ("sddd", 200, 96, 2048, "col"), ("czcs", 77, 200, 40, "col")]


@pytest.fixture(scope="module")
def comm():
    import torch
    torch.cuda.set_device(0)
    c = M.Comm(M.comm_unique_id(), 1, 0)
    yield c
    c.close()


def unsharded(p, alpha, beta, numerics):
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm(alpha, da, db, beta, dc, config({"gpu.numerics": numerics, "gpu.splitk": "off"}))
    return dC.bytes()


def col_slice(v, j0, nb):
    out = v.copy()
    out.base = v.base + j0 * v.cs * M.dtype_size(v.dtype)
    out.n = nb
    return out


@pytest.mark.parametrize("label,m,n,k,kind", CASES)
@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("numerics", ["fast", "exact"])
def test_sharded_panels_equal_unsharded(comm, label, m, n, k, kind, world, numerics):
    import torch
    p = Problem(label, m, n, k, c_kind=kind, seed=9)
    cid = M.CaseLabel.parse(label).case_id()
    alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
    want = unsharded(p, alpha, SCALARS["cfg2_beta"], numerics)
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    flops = 0
    for r in range(world):
        j0, nb = M.shard_columns(n, world, r, 64)
        if nb == 0:
            continue
        flops += M.gemm_sharded(comm, 0, alpha, da, col_slice(db, j0, nb), SCALARS["cfg2_beta"], col_slice(dc, j0, nb),
                                config({"gpu.numerics": numerics}))
    torch.cuda.synchronize()
    assert flops > 0
    assert np.array_equal(dC.bytes(), want), (label, world)


def test_sharded_whole_problem_and_bad_root(comm):
    # one rank owning every column is the plain call; a root outside the communicator is an Error
    import torch
    p = Problem("dzzd", 50, 60, 70, seed=2)
    want = unsharded(p, SCALARS["p7"], SCALARS["one"], "fast")
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    M.gemm_sharded(comm, 0, SCALARS["p7"], da, db, SCALARS["one"], dc, config({"gpu.numerics": "fast"}))
    torch.cuda.synchronize()
    assert np.array_equal(dC.bytes(), want)
    with pytest.raises(M.Error):
        M.gemm_sharded(comm, 1, SCALARS["p7"], da, db, SCALARS["one"], dc)  # no rank 1


@pytest.mark.parametrize("where", ["device", "host"])
def test_gemm_multi_one_device(where):
    for label, m, n, k, kind in CASES:
        p = Problem(label, m, n, k, c_kind=kind, seed=4)
        cid = M.CaseLabel.parse(label).case_id()
        alpha = SCALARS["cfg3_alpha"] if cid == 7 else SCALARS["p7"]
        want = unsharded(p, alpha, SCALARS["cfg2_beta"], "fast")
        if where == "device":
            dA, dB, dC = p.device()
            da, db, dc = p.views(A=dA, B=dB, C=dC)
            M.gemm_multi(alpha, da, db, SCALARS["cfg2_beta"], dc, config({"gpu.numerics": "fast"}), devices=[0])
            got = dC.bytes()
        else:
            out = p.C.clone()
            va, vb, vc = p.views(C=out)
            M.gemm_multi(alpha, va, vb, SCALARS["cfg2_beta"], vc, config({"gpu.numerics": "fast"}), devices=[0])
            got = out.buf
        assert np.array_equal(got, want), (label, where)


def test_gemm_multi_rejects_missing_devices_and_policy_errors():
    p = Problem("zddd", 8, 8, 8)
    dA, dB, dC = p.device()
    da, db, dc = p.views(A=dA, B=dB, C=dC)
    import torch
    with pytest.raises(M.Error):
        M.gemm_multi(SCALARS["p7"], da, db, SCALARS["one"], dc, devices=[torch.cuda.device_count()])
    with pytest.raises(M.ScalarPolicyError):
        M.gemm_multi(SCALARS["c55"], da, db, SCALARS["one"], dc, devices=[0])
