"""Isolated call rate of one label at m=n=k=s for several betas (and alpha
per case), classic vs MDGEMM_DMMA_WS (set outside)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06015_b200 as M
from tests.test_baseline_scale_gpu import DevMat
from tests.helpers import config

lab = sys.argv[1]
s = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
A, B, C = DevMat(da, s, s, 1), DevMat(db, s, s, 2), DevMat(dc, s, s, 3)
cid = M.CaseLabel.parse(lab).case_id()
alpha = M.Scalar.complex_value(1.2, -0.7) if cid in (0, 7) else M.Scalar.real_value(1.2)
cfg = config({})
for name, beta in (("beta=0", M.Scalar.real_value(0.0)), ("beta=1", M.Scalar.real_value(1.0)),
                   ("beta=0.9+0.3i", M.Scalar.complex_value(0.9, 0.3))):
    call = lambda: M.gemm_async(alpha, A.view(), B.view(), beta, C.view(comp), cfg)
    call(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): call()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(lab, s, name, f"{ms:.3f} ms", f"{M.flops_of_case(cid, s, s, s) / ms / 1e9:.1f} TF/s")
