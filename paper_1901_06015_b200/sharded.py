"""Column-panel split of one gemm over the ranks of a process group.

C and B are divided into column panels (mdg_shard_columns: equal panels,
multiples of `align` columns, the last one shorter); every rank runs an
independent gemm on slice(B, 0, j0, k, nb) and slice(C, 0, j0, m, nb)
(dtypes.cpp:157-166) with the whole of A, which rank 0 broadcasts.  No
reduction is needed: each C element belongs to exactly one rank.  The
per-element accumulation order does not depend on the tile a column lands
in, so every shard is bitwise identical to the same columns of the unsharded
run in EXACT numerics, and in FAST numerics whenever the unsharded call does
not take split-K (a shard never does; gpu.splitk = off keeps any call on the
whole-k grid).

On GPUs the library does the whole exchange (mdg_gemm_sharded through a
library communicator, `comm`): A is broadcast with NCCL over NVLink/NVSwitch
on a side stream while the rank packs its B panel.  Without a communicator
(the CPU tests: gloo), A travels as raw bytes through
torch.distributed.broadcast.  The column slicing works on the ORIGINAL C, so
plans that transpose the operation (row-stored C, case 2bc) shard exactly the
same way.
"""
from __future__ import annotations

from typing import Callable, Optional

import paper_1901_06015_b200 as M

DEFAULT_ALIGN = 128  # a CTA tile of the fast kernels


def column_panel(n: int, world: int, rank: int, align: int = DEFAULT_ALIGN) -> tuple[int, int]:
    """[j0, j0 + nb) of the n columns owned by `rank`."""
    return M.shard_columns(n, world, rank, align)


def slice_columns(v: "M.MatrixView", j0: int, nb: int) -> "M.MatrixView":
    """slice(v, 0, j0, v.m, nb) without validation of an empty window."""
    if j0 < 0 or nb < 0 or j0 + nb > v.n:
        raise M.Error("slice: window out of range")
    out = v.copy()
    out.base = (v.base or 0) + j0 * v.cs * M.dtype_size(v.dtype)
    out.n = nb
    return out


def gemm_sharded(alpha, a: "M.MatrixView", b: "M.MatrixView", beta, c: "M.MatrixView", cfg=None, *,
                 world: int = 1, rank: int = 0, group=None, a_bytes=None, align: int = DEFAULT_ALIGN,
                 stream=None, compute: Optional[Callable] = None, comm: "Optional[M.Comm]" = None) -> int:
    """Run rank `rank`'s share of C := beta*C + alpha*A*B.

    `a`, `b`, `c` describe the FULL operands as seen by this rank; only the
    columns [j0, j0+nb) of `b` and `c` are touched.  `a_bytes` (a torch
    tensor aliasing A's storage) is broadcast from rank 0 first when world > 1.
    `compute(alpha, a, b, beta, c, cfg, stream)` defaults to the device gemm
    (gemm_async on `stream`); tests substitute the CPU oracle.  Returns the
    FlopCounter value of the local share.  With `comm` (a library
    communicator, one process per GPU) the library broadcasts A itself."""
    if comm is not None:
        j0, nb = column_panel(c.n, comm.nranks, comm.rank, align)
        return M.gemm_sharded(comm, 0, alpha, a, slice_columns(b, j0, nb), beta, slice_columns(c, j0, nb), cfg,
                              stream)
    if world > 1 and a_bytes is not None:
        import torch.distributed as dist
        dist.broadcast(a_bytes, src=0, group=group)
    j0, nb = column_panel(c.n, world, rank, align)
    if nb == 0:
        return 0
    bl, cl = slice_columns(b, j0, nb), slice_columns(c, j0, nb)
    if compute is None:
        return M.gemm_async(alpha, a, bl, beta, cl, cfg, stream)
    return compute(alpha, a, bl, beta, cl, cfg, stream)
