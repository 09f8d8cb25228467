"""World-size-2 gloo run of the column-panel split on CPU:
rank 0 owns A and broadcasts it, each rank computes its column panel of C
(through the oracle standing in for the device gemm), rank 0 gathers the
panels and checks them bitwise against the unsharded result, for every
domain case, row-stored C (the transposed plans) and odd splits."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1901_06015_b200 as M
from oracle import oracle as O
from paper_1901_06015_b200.sharded import column_panel, gemm_sharded
from tests.helpers import Problem, SCALARS

CASES = [("dddd", 37, 45, 29, "col", 8), ("zzzd", 20, 33, 17, "col", 8), ("cdds", 16, 40, 300, "col", 16),
         ("zdzs", 19, 26, 21, "row", 4), ("sccs", 12, 17, 9, "gen", 2), ("ccsd", 14, 10, 30, "col", 1)]


def _oracle_compute(alpha, a, b, beta, c, cfg, stream):
    return O.orc_gemm(alpha, a, b, beta, c, cfg)


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for label, m, n, k, kind, align in CASES:
            p = Problem(label, m, n, k, c_kind=kind, seed=5)
            if rank != 0:
                p.A.buf[:] = 0  # only rank 0 holds A before the broadcast
            a_bytes = torch.from_numpy(p.A.buf)
            va, vb, vc = p.views()
            flops = gemm_sharded(SCALARS["p7"], va, vb, SCALARS["c34"], vc, M.Config.defaults(), world=world,
                                 rank=rank, a_bytes=a_bytes, align=align, compute=_oracle_compute)
            mine = torch.from_numpy(p.C.buf.copy())
            gathered = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
            dist.gather(mine, gathered, dst=0)
            ftot = torch.tensor([flops], dtype=torch.int64)
            dist.all_reduce(ftot)
            if rank == 0:
                ref = Problem(label, m, n, k, c_kind=kind, seed=5)
                ra, rb, rc = ref.views()
                O.orc_gemm(SCALARS["p7"], ra, rb, SCALARS["c34"], rc)
                merged = ref.C.clone()
                for r in range(world):
                    j0, nb = column_panel(n, world, r, align)
                    part = p.C.clone()
                    part.buf[:] = gathered[r].numpy()
                    merged.values()[:, j0:j0 + nb] = part.values()[:, j0:j0 + nb]
                results[label] = (merged.buf.tobytes() == ref.C.buf.tobytes(), int(ftot.item()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_column_panels_gloo(world):
    results = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert set(results.keys()) == {c[0] for c in CASES}
    for label, (ok, flops) in results.items():
        assert ok, f"{label}: sharded result differs from the unsharded run"
        assert flops > 0


def test_panels_cover_columns():
    for n in (1, 7, 128, 1000, 16384):
        for world in (1, 2, 4, 8):
            seen = np.zeros(n, int)
            for r in range(world):
                j0, nb = column_panel(n, world, r, 128)
                seen[j0:j0 + nb] += 1
            assert np.all(seen == 1)
