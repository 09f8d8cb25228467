import os, sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_1901_06015_b200 as M
from tests.test_baseline_scale_gpu import DevMat
from tests.helpers import config
for (label, m, n, k) in [("dddd", 256, 256, 16384), ("ssss", 256, 256, 16384), ("zzzd", 128, 256, 8192), ("dddd", 512, 512, 512), ("dddd", 1024, 1024, 1024)]:
    dc, da, db = (M.dtype_from_letter(ch) for ch in label[:3]); comp = M.SINGLE if label[3] == "s" else M.DOUBLE
    A = DevMat(da, m, k, 1); B = DevMat(db, k, n, 2); C = DevMat(dc, m, n, 3)
    res = []
    for sk in ["1", "0"]:
        os.environ["MDGEMM_SPLITK"] = sk
        cfg = config({})
        for _ in range(3): M.gemm_async(M.Scalar.real_value(1.0), A.view(), B.view(), M.Scalar.real_value(1.0), C.view(comp), cfg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): M.gemm_async(M.Scalar.real_value(1.0), A.view(), B.view(), M.Scalar.real_value(1.0), C.view(comp), cfg)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl = M.flops_of_case(M.CaseLabel.parse(label).case_id(), m, n, k)
        res.append(f"split={'off' if sk == '1' else 'auto'} {fl / ms / 1e9:.1f} TF")
    print(label, m, n, k, res)
