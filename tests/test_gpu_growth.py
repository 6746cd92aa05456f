"""NEXT-2: cell growth and division on the GPU against the oracle.
The paper's first GPU benchmark ("cell growth and division", 1.27x on a
V100).  Population, ids, positions, diameters and the last mechanics displacements must equal the
oracle bit for bit after several steps with growth, divisions and capacity reallocations."""
import numpy as np
import pytest

import bdm_inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bdm():
    import torch

    assert torch.cuda.is_available()
    import paper_2006_06775_b200 as b

    return b


def gpu_run(bdm, pos, diam, steps, growth, div, seed, **kw):
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(**kw))
    bdm.bdm_set_growth(h, growth, div, seed)
    bdm.bdm_mech_step(h, steps)
    return h, bdm.bdm_get_positions(h), bdm.bdm_get_diameters(h), bdm.bdm_get_displacements(h)


@pytest.mark.parametrize("steps", [1, 3, 8])
def test_growth_division_parity(bdm, steps):
    pos, diam = bdm_inputs.random_instance(21, 3000, 220.0, 8.0, 12.0)
    h, p, d, dp = gpu_run(bdm, pos, diam, steps, 0.6, 12.0, 77)
    po, do, dpo = oracle.run_growth(pos, diam, steps, 0.6, 12.0, 77)
    assert len(d) == len(do) > len(diam)
    assert np.array_equal(d, do)
    assert np.array_equal(p, po)
    n_dp = bdm.bdm_get_count(h)[1]
    assert np.array_equal(dp, dpo[:n_dp])


def test_doubling_and_capacity_growth(bdm):
    """SPEC.md:101 doubling oracle on the GPU: every agent divides every step; 7 steps take 20
    agents to 2560 through several capacity reallocations."""
    pos, diam = bdm_inputs.random_instance(5, 20, 400.0, 9.0, 10.0)
    h, p, d, _ = gpu_run(bdm, pos, diam, 7, 0.0, 1.0, 3)
    assert len(d) == 20 * 2 ** 7
    po, do, _ = oracle.run_growth(pos, diam, 7, 0.0, 1.0, 3)
    assert np.array_equal(p, po) and np.array_equal(d, do)


def test_growth_changes_box_edge(bdm):
    """O1 after growth: the box edge follows the largest diameter of the new population."""
    pos, diam = bdm_inputs.random_instance(9, 500, 150.0, 8.0, 10.0)
    h, p, d, _ = gpu_run(bdm, pos, diam, 2, 1.5, 50.0, 1)
    bdm.bdm_grid_build(h)
    assert bdm.bdm_get_grid_info(h)["L"] == d.max() == diam.max() + 3.0


def test_growth_large_dense_population(bdm):
    """1.5e6 agents at the density of cfg2 (fewer boxes than agents, so the division-rank scan
    needs more tiles than the box-table scan): 2 steps against the oracle, bit for bit."""
    n = 1_500_000
    side = (n / 1e-3) ** (1.0 / 3.0)
    pos, diam = bdm_inputs.uniform_population(6, np.arange(n), (0.0, 0.0, 0.0), (side, side, side), 8.0, 12.0)
    h, p, d, dp = gpu_run(bdm, pos, diam, 2, 0.8, 12.0, 6)
    po, do, dpo = oracle.run_growth(pos, diam, 2, 0.8, 12.0, 6, cap=4 * n)
    assert len(d) == len(do) > n
    assert np.array_equal(d, do) and np.array_equal(p, po)
