#!/usr/bin/env python3
"""Regenerates tests/golden/reference_vectors.json from the REFERENCE engine
itself (oracle/_ref/libmdgemm_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Each record names a seeded problem (inputs are re-drawn
from the reference Rng, so only the recipe is stored) and the SHA-256 of the
bytes the reference produced: C after gemm() (gaps of general storage
included) or the packed buffer of pack_block().  Run here, where the
reference sources exist; the JSON is committed and travels to the GPU box.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1901_06015_b200 as M  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.helpers import ALL_LABELS, HostMatrix, Problem, SCALARS, config  # noqa: E402

GEMM_SPECS = []
for i, label in enumerate(ALL_LABELS):
    GEMM_SPECS.append(dict(label=label, m=17, n=16, k=19, kind="col", trans_a=False, trans_b=False, conj_a=False,
                           conj_b=False, alpha="p7", beta="m3", cfg={}))
    GEMM_SPECS.append(dict(label=label, m=13, n=7, k=19, kind=["row", "gen", "col"][i % 3], trans_a=i % 2 == 0,
                           trans_b=i % 3 == 0, conj_a=True, conj_b=i % 4 == 0,
                           alpha="cfg2_alpha_real", beta="cfg2_beta",
                           cfg=[{}, {"ctemp.enable": "off", "gemm.kc": "8"}, {"ukr.preference": "row"},
                                {"gemm.threads": "4"}][i % 4]))
    cid = M.CaseLabel.parse(label).case_id()
    if cid in (0, 7):
        GEMM_SPECS.append(dict(label=label, m=9, n=11, k=40, kind="col", trans_a=False, trans_b=False,
                               conj_a=False, conj_b=False, alpha="cfg2_alpha", beta="one",
                               cfg={"gemm.kc": "16", "ctemp.enable": "off"}))

PACK_SPECS = []
for dt in range(4):
    for side in (M.LEFT, M.RIGHT):
        for fmt in ((M.STANDARD, M.ONE_E, M.ONE_R) if M.is_complex(dt) else (M.STANDARD,)):
            for tp in (M.SINGLE, M.DOUBLE):
                target = (2 if M.is_complex(dt) and fmt == M.STANDARD else 0) + tp
                for scale in (("one", "cfg3_alpha") if fmt != M.STANDARD else ("one", "minus_one")):
                    PACK_SPECS.append(dict(dtype=dt, m=6, n=5, kind="gen", side=side, fmt=fmt, conj=1, src_conj=0,
                                           scale=scale, target=target, reg_block=4))


def run_gemm(spec, fn):
    p = Problem(spec["label"], spec["m"], spec["n"], spec["k"], c_kind=spec["kind"], trans_a=spec["trans_a"],
                trans_b=spec["trans_b"], conj_a=spec["conj_a"], conj_b=spec["conj_b"], seed=2024)
    va, vb, vc = p.views()
    flops = fn(SCALARS[spec["alpha"]], va, vb, SCALARS[spec["beta"]], vc, config(spec["cfg"]))
    return hashlib.sha256(p.C.buf.tobytes()).hexdigest(), flops


def pack_input(spec):
    return HostMatrix(spec["dtype"], spec["m"], spec["n"], spec["kind"]).fill(O.orc_rng_state(2024, ["golden-pack"]))


def main():
    if O.ref is None:
        sys.exit("oracle/_ref is not built; run `make -C oracle ref` where /root/reference exists")
    gemm = []
    for spec in GEMM_SPECS:
        digest, flops = run_gemm(spec, O.ref_gemm)
        gemm.append({**spec, "sha256": digest, "flops": flops})
    pack = []
    for spec in PACK_SPECS:
        src = pack_input(spec)
        v = src.view(conj=bool(spec["src_conj"]))
        n = O.ref_packed_bytes(v, spec["side"], spec["fmt"], spec["target"], spec["reg_block"])
        buf = np.zeros(n, np.uint8)
        O.ref_pack(v, spec["side"], spec["fmt"], spec["conj"], SCALARS[spec["scale"]], spec["target"],
                   spec["reg_block"], buf.ctypes.data, n)
        pack.append({**spec, "bytes": int(n), "sha256": hashlib.sha256(buf.tobytes()).hexdigest()})
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref (reference sources, -O3 -DNDEBUG)",
           "seed": 2024, "gemm": gemm, "pack": pack}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {len(gemm)} gemm and {len(pack)} pack vectors to {path}")


if __name__ == "__main__":
    main()
