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
