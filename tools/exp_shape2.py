"""Like exp_shape.py with beta given: lab m n k beta_re beta_im"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06015_b200 as M
from tests.test_baseline_scale_gpu import DevMat
from tests.helpers import config
lab, m, n, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
br, bi = float(sys.argv[5]), float(sys.argv[6])
dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
A, B, C = DevMat(da, m, k, 1), DevMat(db, k, n, 2), DevMat(dc, m, n, 3)
cid = M.CaseLabel.parse(lab).case_id()
alpha = M.Scalar.complex_value(1.2, -0.7) if cid in (0, 7) else M.Scalar.real_value(1.2)
beta = M.Scalar.complex_value(br, bi) if bi else M.Scalar.real_value(br)
cfg = config({})
call = lambda: M.gemm_async(alpha, A.view(), B.view(), beta, C.view(comp), cfg)
call(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(3): call()
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 3
print(lab, m, n, k, br, bi, os.environ.get("MDGEMM_DMMA_WS"), os.environ.get("MDGEMM_STREAMK"), f"{ms:.3f} ms", f"{M.flops_of_case(cid, m, n, k) / ms / 1e9:.1f} TF/s")
