"""Device input generator vs the reference Rng/fill_uniform (rng.hpp:13-56):
bitwise, so GPU-resident benchmark operands equal the CPU ones."""
import pytest

import paper_1901_06015_b200 as M
from oracle import oracle as O
from tests.helpers import ALL_DT, HostMatrix

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ALL_DT)
@pytest.mark.parametrize("kind", ["col", "row", "gen"])
def test_fill_uniform_bitwise(dtype, kind):
    state = M.Rng(0).split("zzzd").split("bench").split("a").state
    assert state == O.orc_rng_state(0, ["zzzd", "bench", "a"])
    host = HostMatrix(dtype, 37, 29, kind).fill(state)
    dev = HostMatrix(dtype, 37, 29, kind).to_device()
    M.fill_uniform(dev.view(), state)
    assert dev.bytes().tobytes() == host.buf.tobytes()


@pytest.mark.parametrize("dtype", ALL_DT)
def test_fill_normal_box_muller_of_the_reference_draws(dtype):
    # mdg_fill_normal: Box-Muller over the reference Rng's draws 2t, 2t+1 (BASELINE configs[4]
    # asks for normal(0,1) entries and the reference has no normal generator).  The numpy
    # restatement uses the host libm: equal up to a few ulp of the device's log / cospi.
    import numpy as np
    state = M.Rng(0).split("cfg5").split("normal").state
    m, n = 301, 77
    dev = HostMatrix(dtype, m, n).to_device()
    M.fill_normal(dev.view(), state)
    h = HostMatrix(dtype, m, n)
    h.buf[:] = dev.bytes()
    vals = h.values().T.reshape(-1)  # draw order: column-major, re then im
    comps = np.stack([vals.real, vals.imag], 1).reshape(-1) if M.is_complex(dtype) else vals.real
    want = O.normal_values(state, np.arange(comps.size))
    if M.precision_of(dtype) == M.SINGLE:
        want = want.astype(np.float32).astype(np.float64)
        tol = 4 * 2.0 ** -24
    else:
        tol = 64 * 2.0 ** -53
    assert np.all(np.abs(comps - want) <= tol * np.maximum(np.abs(want), 1.0))
    big = HostMatrix(M.DT_D, 1 << 20, 1).to_device()
    M.fill_normal(big.view(), state)
    z = big.bytes().view(np.float64)
    assert abs(z.mean()) < 5e-3 and abs(z.std() - 1.0) < 5e-3
