"""Fused column pass: the sum pass accumulates the next build's column z-ranges in
the frame (step-start extents +- 1 box).  Multi-step trajectories must stay bit-equal to the oracle
with and without the fusion (max_disp >= L disables it), grid info must report the tight extents,
and a new population (bdm_set_agents) must not reuse stale columns."""
import numpy as np
import pytest

import bdm_inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bdm():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2006_06775_b200 as b

    b.load_library()
    return b


def trajectory(bdm, pos, diam, steps, **kw):
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(**kw))
    for _ in range(steps):
        bdm.bdm_mech_step(h, 1)
    return h, bdm.bdm_get_positions(h)


@pytest.mark.parametrize("max_disp", [3.0, 11.0, 30.0])  # fused, fused (close to L), not fused (>= L)
def test_multistep_bit_exact(bdm, max_disp):
    rng = np.random.default_rng(5)
    n = 5000
    pos = rng.uniform(0, 180, (n, 3))
    diam = rng.uniform(8, 12, n)
    h, p = trajectory(bdm, pos, diam, 5, max_disp=max_disp)
    ref, _ = oracle.run(pos, diam, 5, oracle.params(max_disp=max_disp))
    assert np.array_equal(p, ref)
    info = bdm.bdm_get_grid_info(h)
    bdm.bdm_grid_build(h)  # grid of the current positions (fused frame if the last step fused it)
    info = bdm.bdm_get_grid_info(h)
    gp = oracle.grid_params(ref, diam)
    assert info["lo"] == gp["lo"] and info["hi"] == gp["hi"]  # tight extents reported
    assert np.array_equal(bdm.bdm_get_box_coords(h), oracle.box_coords(ref, diam))


def test_pairs_after_fused_steps(bdm):
    pos, diam = bdm_inputs.make_config(1)
    h, p = trajectory(bdm, pos, diam, 3)
    for kind in (0, 1):
        assert np.array_equal(bdm.bdm_get_pairs(h, kind), oracle.pairs(p, diam, kind))


def test_set_agents_after_fused_steps(bdm):
    rng = np.random.default_rng(9)
    n = 3000
    pos = rng.uniform(0, 150, (n, 3))
    diam = rng.uniform(8, 12, n)
    h, _ = trajectory(bdm, pos, diam, 2)
    pos2 = rng.uniform(-400, -250, (n, 3))  # a different region: stale columns would be wrong
    bdm.bdm_set_agents(h, pos2, diam)
    bdm.bdm_mech_step(h, 2)
    ref, _ = oracle.run(pos2, diam, 2)
    assert np.array_equal(bdm.bdm_get_positions(h), ref)


@pytest.mark.parametrize("max_disp", [3.0, 11.0])
def test_deferred_builds_bit_exact(bdm, max_disp):
    """One bdm_mech_step(12) call defers the builds of steps 0..10 (no host round trip: the grid is
    the fused frame, growing one box per axis per step, re-tightened after 8) -- positions equal the
    oracle's and those of 12 single-step calls (every build synchronised); grid info stays tight."""
    rng = np.random.default_rng(8)
    n = 6000
    pos = rng.normal(0.0, 40.0, (n, 3))
    diam = np.clip(rng.lognormal(np.log(10.0), 0.15, n), 6.0, 16.0)
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(max_disp=max_disp))
    bdm.bdm_set_defer(h, 8)
    bdm.bdm_mech_step(h, 12)
    p = bdm.bdm_get_positions(h)
    _, p1 = trajectory(bdm, pos, diam, 12, max_disp=max_disp)
    assert np.array_equal(p, p1)
    ref, _ = oracle.run(pos, diam, 12, oracle.params(max_disp=max_disp))
    assert np.array_equal(p, ref)
    # grid info describes the last step's build: the tight extents of its start positions
    start11, _ = oracle.run(pos, diam, 11, oracle.params(max_disp=max_disp))
    gp = oracle.grid_params(start11, diam)
    info = bdm.bdm_get_grid_info(h)
    assert info["lo"] == gp["lo"] and info["hi"] == gp["hi"]
