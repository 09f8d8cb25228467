"""Short-k epilogue cost: the same sddd rank-64 update with beta = 0 (no C
read), 1 and a general real beta, device-resident, CUDA events."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06015_b200 as M
from tests.test_baseline_scale_gpu import DevMat
from tests.helpers import config

lab = sys.argv[1] if len(sys.argv) > 1 else "sddd"
m = n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
k = int(sys.argv[3]) if len(sys.argv) > 3 else 64
dc, da, db = (M.dtype_from_letter(ch) for ch in lab[:3])
comp = M.SINGLE if lab[3] == "s" else M.DOUBLE
A, B, C = DevMat(da, m, k, 1), DevMat(db, k, n, 2), DevMat(dc, m, n, 3)
cfg = config({})
for name, beta in (("beta=0", M.Scalar.real_value(0.0)), ("beta=1", M.Scalar.real_value(1.0)), ("beta=0.9", M.Scalar.real_value(0.9))):
    call = lambda: M.gemm_async(M.Scalar.real_value(-1.0), A.view(), B.view(), beta, C.view(comp), cfg)
    call(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): call()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(lab, m, n, k, name, f"{ms:.3f} ms", f"{2.0 * m * n * k / ms / 1e9:.1f} TF/s")
