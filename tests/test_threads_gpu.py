"""gemm() is reentrant, like the reference's (SPEC: no globals, exclusive C):
host threads calling it at the same time on their own operands -- device
operands (the lone-call path on the legacy stream), pageable host operands
(the batch runner, the library's streams and its pinned staging ring) and
batches -- must each get exactly the bits a sequential call gives.  (ctypes
releases the GIL around every library call, so the threads really overlap.)"""
import threading

import pytest

import paper_1901_06015_b200 as M
from tests.helpers import Problem, SCALARS, config

pytestmark = pytest.mark.gpu

FAST = config({"gpu.numerics": "fast"})
LABELS = ["dddd", "zzzd", "cdds", "sddd", "cccs", "szzs", "zczd", "dssd"]


def problems(seed):
    # host windows above the pinned ring's direct-copy threshold (1 MB) for half of them
    return [Problem(l, 300 + 40 * (i % 3), 280, 200 + 64 * (i % 2), seed=seed + i) for i, l in enumerate(LABELS)]


def run_threads(fn, n):
    errors = []

    def wrap(t):
        try:
            fn(t)
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=wrap, args=(t,)) for t in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("where", ["device", "host"])
def test_concurrent_gemm_calls(where):
    probs = problems(500)
    # sequential reference (device operands)
    want = []
    for p in probs:
        dA, dB, dC = p.device()
        da, db, dc = p.views(A=dA, B=dB, C=dC)
        M.gemm(SCALARS["p7"], da, db, SCALARS["cfg2_beta"], dc, FAST)
        want.append(dC.bytes().tobytes())
    got = [None] * len(probs)
    if where == "device":
        devs = [p.device() for p in probs]

        def work(t):
            for rep in range(3):
                for i in range(t, len(probs), 4):
                    p = probs[i]
                    dA, dB, _ = devs[i]
                    dC = p.C.to_device()
                    da, db, dc = p.views(A=dA, B=dB, C=dC)
                    M.gemm(SCALARS["p7"], da, db, SCALARS["cfg2_beta"], dc, FAST)
                    got[i] = dC.bytes().tobytes()
    else:
        def work(t):
            for rep in range(3):
                for i in range(t, len(probs), 4):
                    p = probs[i]
                    c = p.C.clone()
                    va, vb, vc = p.views(C=c)
                    M.gemm(SCALARS["p7"], va, vb, SCALARS["cfg2_beta"], vc, FAST)
                    got[i] = c.buf.tobytes()
    run_threads(work, 4)
    for i, p in enumerate(probs):
        assert got[i] == want[i], (where, p.label)


def test_concurrent_batches():
    probs = problems(700)
    want = []
    for p in probs:
        c = p.C.clone()
        va, vb, vc = p.views(C=c)
        M.gemm(SCALARS["m3"], va, vb, SCALARS["one"], vc, FAST)
        want.append(c.buf.tobytes())
    outs = {}

    def work(t):
        cs = [p.C.clone() for p in probs]
        calls = []
        for p, c in zip(probs, cs):
            va, vb, vc = p.views(C=c)
            calls.append((SCALARS["m3"], va, vb, SCALARS["one"], vc))
        M.gemm_batch(calls, FAST)
        outs[t] = [c.buf.tobytes() for c in cs]

    run_threads(work, 3)
    for t in range(3):
        assert outs[t] == want, t
