"""Device pack kernels vs the oracle pack (itself pinned bitwise to the
reference pack_block, test_oracle_pins.py): byte-for-byte, signed zeros
included.  Reference KATs: test_packing.cpp:27-253."""
import itertools

import numpy as np
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import ALL_DT, HostMatrix, SCALARS

pytestmark = pytest.mark.gpu


def _device_pack(src: HostMatrix, side, fmt, conj, scale, target, rb, plen=0, src_conj=False):
    import torch
    d = src.to_device()
    v = d.view(conj=src_conj)
    nbytes = M.packed_bytes(v, side, fmt, target, rb, plen)
    out = torch.full((nbytes,), 0x5A, dtype=torch.uint8, device="cuda")
    M.pack_block_device(out.data_ptr(), v, side, fmt, conj, scale, target, rb, plen)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _oracle_pack(src: HostMatrix, side, fmt, conj, scale, target, rb, plen=0, src_conj=False):
    v = src.view(conj=src_conj)
    nbytes = O.orc_packed_bytes(v, side, fmt, target, rb, plen)
    out = np.full(nbytes, 0xA5, np.uint8)
    O.orc_pack(v, side, fmt, conj, scale, target, rb, plen, out.ctypes.data)
    return out


def _cases():
    for dt, side, fmt, conj in itertools.product(ALL_DT, (M.LEFT, M.RIGHT), (M.STANDARD, M.ONE_E, M.ONE_R), (0, 1)):
        if fmt != M.STANDARD and not M.is_complex(dt):
            continue
        for tp in (M.SINGLE, M.DOUBLE):
            target = (2 if (M.is_complex(dt) and fmt == M.STANDARD) else 0) + tp
            yield dt, side, fmt, conj, target


@pytest.mark.parametrize("dt,side,fmt,conj,target", list(_cases()))
def test_pack_bitwise(dt, side, fmt, conj, target):
    scales = ["one", "p7", "minus_one"] + ([] if fmt == M.STANDARD else ["cfg3_alpha"])
    for (m, n), kind, rb, plen, sc, src_conj in itertools.product(
            [(5, 7), (33, 70), (130, 3)], ["col", "row", "gen"], [2, 4, 64], [0, 1], scales, [False, True]):
        if fmt != M.ONE_E and rb == 2:
            rb = 3  # odd panel dims are legal for Standard/1r
        src = HostMatrix(dt, m, n, kind).fill(O.orc_rng_state(11, ["pack", dt, kind, m]))
        if plen:  # zero-padded inner dimension, longer than any logical panel
            plen = 2 * max(m, n) + 16
        args = (side, fmt, conj, SCALARS[sc], target, rb, plen)
        got = _device_pack(src, *args, src_conj=src_conj and M.is_complex(dt))
        want = _oracle_pack(src, *args, src_conj=src_conj and M.is_complex(dt))
        assert got.tobytes() == want.tobytes(), (m, n, kind, rb, plen, sc, src_conj)


def test_kat_one_e_left():
    # test_packing.cpp:27-38: [3+4i] -> [[3,-4],[4,3]]
    a = HostMatrix(M.DT_Z, 1, 1)
    a.values()[0, 0] = 3 + 4j
    got = _device_pack(a, M.LEFT, M.ONE_E, 0, SCALARS["one"], M.DT_Z, 2).view(np.float64)
    # left panel, column-major within the panel: (0,0),(1,0),(0,1),(1,1)
    assert list(got) == [3.0, 4.0, -4.0, 3.0]


def test_kat_conj_one_r_right():
    # test_packing.cpp:40-48: conj 1r right [5+6i] -> [5; -6]
    b = HostMatrix(M.DT_Z, 1, 1)
    b.values()[0, 0] = 5 + 6j
    got = _device_pack(b, M.RIGHT, M.ONE_R, 1, SCALARS["one"], M.DT_Z, 2).view(np.float64)
    # right panel of 2 columns: row 0 = (5, pad), row 1 = (-6, pad)
    assert got[0] == 5.0 and got[2] == -6.0 and got[1] == 0.0 and got[3] == 0.0


def test_negative_zero_in_one_e_padding():
    # padded complex slots write -0.0 into the -Im position (packing.cpp:189-191)
    a = HostMatrix(M.DT_Z, 1, 1)
    a.values()[0, 0] = 1 + 1j
    got = _device_pack(a, M.LEFT, M.ONE_E, 0, SCALARS["one"], M.DT_D, 4).view(np.float64)
    # panel of 4 real rows: rows 2,3 pad; column 1 holds (-im, re) pairs -> row 2 is -0.0
    col1 = got[4:8]
    assert np.signbit(col1[2]) and col1[2] == 0.0 and not np.signbit(col1[3])


def test_pack_errors_surface_as_error():
    import torch
    src = HostMatrix(M.DT_D, 2, 2).fill(1).to_device()
    buf = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    with pytest.raises(M.Error):
        M.pack_block_device(buf.data_ptr(), src.view(), M.LEFT, M.ONE_E, 0, SCALARS["one"], M.DT_D, 4)
    zsrc = HostMatrix(M.DT_Z, 2, 2).fill(1).to_device()
    with pytest.raises(M.Error):
        M.pack_block_device(buf.data_ptr(), zsrc.view(), M.LEFT, M.STANDARD, 0, SCALARS["c55"], M.DT_Z, 4)


@pytest.mark.parametrize("dt", [M.DT_S, M.DT_D])
@pytest.mark.parametrize("side", [M.LEFT, M.RIGHT])
@pytest.mark.parametrize("tp", [M.SINGLE, M.DOUBLE])
def test_pack_vector_tiles(dt, side, tp):
    """Real sources with a unit-stride axis and 16-byte aligned lines take the vector tiles
    (pack_tile.cuh: vec_ok / pack_tile_vec): sub-blocks of a parent matrix whose leading
    dimension is a multiple of four elements, extents that end inside a vector, inside a tile and
    past several tiles, aligned and unaligned origins (the latter fall back to scalar tiles),
    both storage orders (= both the straight and the transposing path per side)."""
    import torch
    es = M.dtype_size(dt)
    for (pm, pn), (m, n), (oi, oj), kind, rb, plen, sc in itertools.product(
            [(48, 80), (260, 300)], [(33, 70), (47, 5), (1, 64), (250, 290)], [(0, 0), (4, 2), (1, 0)],
            ["col", "row"], [4, 64, 128], [0, 1], ["one", "p7"]):
        if oi + m > pm or oj + n > pn:
            continue
        parent = HostMatrix(dt, pm, pn, kind).fill(O.orc_rng_state(13, ["vec", dt, kind, pm]))
        off = (oi * parent.rs + oj * parent.cs) * es
        hv = M.MatrixView.make(parent.buf.ctypes.data + off, m, n, parent.rs, parent.cs, dt)
        dev = torch.from_numpy(parent.buf.copy()).cuda()
        dv = M.MatrixView.make(dev.data_ptr() + off, m, n, parent.rs, parent.cs, dt)
        pl = 2 * max(m, n) + 16 if plen else 0
        nbytes = O.orc_packed_bytes(hv, side, M.STANDARD, tp, rb, pl)
        assert nbytes == M.packed_bytes(dv, side, M.STANDARD, tp, rb, pl)
        want = np.full(nbytes, 0xA5, np.uint8)
        O.orc_pack(hv, side, M.STANDARD, 0, SCALARS[sc], tp, rb, pl, want.ctypes.data)
        out = torch.full((nbytes,), 0x5A, dtype=torch.uint8, device="cuda")
        M.pack_block_device(out.data_ptr(), dv, side, M.STANDARD, 0, SCALARS[sc], tp, rb, pl)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == want.tobytes(), (pm, pn, m, n, oi, oj, kind, rb, plen, sc)
