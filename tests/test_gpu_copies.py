"""Host <-> device state copies at production size: the caller's rows go
through the pinned two-slot ring (64 MB slots) in several chunks, with the
layout conversion (caller pad16 or unpadded rows <-> the device's compact
rows) done by host threads. set_state -> get_state must return the caller's
store bit for bit, padding zeroed (the reference's SolutionStore contract,
solution_store.hpp:16-77)."""
import numpy as np
import pytest

from paper_1208_4772_b200 import mesh as M

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("padded", [True, False])
def test_multi_chunk_roundtrip_bitwise(gpu_lib, padded):
    gpu = gpu_lib
    m = M.cube_mesh(30)  # 162,000 tets: u alone is 32.4M device doubles = 4 ring slots
    fs = gpu.make_state(1.0, [0.3, 0.1, 0.0], 1.0)
    lv = gpu.GpuLevel(m, 4, bc=0, freestream=fs, padded=padded)
    assert lv.K * 5 * lv.device_block > 2 * (8 << 20)
    u = gpu.random_admissible_store(lv, seed=21)
    g = np.random.default_rng(3)
    res = np.where(u != 0.0, g.standard_normal(u.shape), 0.0)
    lv.set_state(u, res)
    u2, r2 = lv.get_state()
    assert np.array_equal(u2, u) and np.array_equal(r2, res)
    if padded:
        pad = u2.reshape(lv.K, 5, lv.block)[:, :, lv.n_basis:]
        assert np.all(pad == 0.0)
    lv.close()
