"""NEXT-1: stationary-region skip -- PAPER.md:454-455 (§2.3(iv) "We detect
stationary regions within the simulation and skip the expensive collision detection for those
agents"), SPEC.md:167-180 (stationary flags), SPEC.md:672 (acceptance #8: a two-cluster scenario
with one frozen cluster stepped 100x with skipping on vs off agrees to 1e-12 per coordinate).

Here the skip is exact by construction, so the tests demand bit equality, and that
the skip really skipped work."""
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


def run(bdm, pos, diam, steps, skip, **kw):
    prm = bdm.bdm_params_default(**kw)
    if skip:
        prm.flags |= bdm.BDM_SKIP_STATIONARY
    h = bdm.bdm_init(pos, diam, prm)
    traj, stats = [], []
    for _ in range(steps):
        bdm.bdm_mech_step(h, 1)
        traj.append(bdm.bdm_get_positions(h))
        stats.append(bdm.bdm_get_skip_stats(h))
    return traj, stats, bdm.bdm_get_displacements(h)


def two_clusters():
    # frozen cluster: simple-cubic lattice of 10 um spheres at 11 um spacing (no contacts)
    g = np.arange(12) * 11.0
    frozen = np.array([(x, y, z) for x in g for y in g for z in g])
    # moving cluster: overlapping random spheres, 10 box lengths away
    rng = np.random.default_rng(8)
    moving = rng.uniform(0.0, 60.0, size=(700, 3)) + np.array([260.0, 0.0, 0.0])
    pos = np.concatenate([frozen, moving])
    diam = np.concatenate([np.full(len(frozen), 10.0), rng.uniform(8.0, 12.0, len(moving))])
    return pos, diam, len(frozen)


def test_two_cluster_skip_bit_identical(bdm):
    """100 steps, skipping on vs off (here: bit for bit)."""
    pos, diam, nf = two_clusters()
    on, st_on, dp_on = run(bdm, pos, diam, 100, True)
    off, _, dp_off = run(bdm, pos, diam, 100, False)
    for s, (a, b) in enumerate(zip(on, off)):
        assert np.array_equal(a, b), f"step {s}"
    assert np.array_equal(dp_on, dp_off)
    # the frozen cluster was skipped: after the first steps far fewer agents are searched than N
    assert st_on[0]["searched"] == len(diam)  # first step: no history, everything searched
    assert max(s["searched"] for s in st_on[5:]) < len(diam) - nf // 2
    # and the frozen cluster really never moved
    assert np.array_equal(on[-1][:nf], pos[:nf])


def test_moving_probe_through_static_lattice(bdm):
    """A jammed pair drifts through a relaxed lattice: agents switch between quiet and hot as the
    disturbance passes (old-box and new-box marking both matter)."""
    g = np.arange(10) * 10.5
    lat = np.array([(x, y, z) for x in g for y in g for z in g])
    probe = np.array([[46.0, 47.0, 47.5], [49.0, 47.5, 47.0], [47.0, 50.0, 46.0]])
    pos = np.concatenate([lat, probe])
    diam = np.concatenate([np.full(len(lat), 10.0), np.array([12.0, 12.0, 12.0])])
    on, st, _ = run(bdm, pos, diam, 60, True, dt=0.3)
    off, _, _ = run(bdm, pos, diam, 60, False, dt=0.3)
    for s, (a, b) in enumerate(zip(on, off)):
        assert np.array_equal(a, b), f"step {s}"
    assert min(x["searched"] for x in st[2:]) < len(diam)  # some steps skipped agents


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_relaxing_population(bdm, seed):
    """Random overlapping population relaxing under adherence: skip on == skip off every step, and
    the skip path matches the oracle trajectory."""
    pos, diam = bdm_inputs.random_instance(300 + seed, 3000, 200.0, 6.0, 12.0)
    on, st, _ = run(bdm, pos, diam, 40, True, adherence=0.5)
    off, _, _ = run(bdm, pos, diam, 40, False, adherence=0.5)
    for s, (a, b) in enumerate(zip(on, off)):
        assert np.array_equal(a, b), f"step {s}"
    ref, _ = oracle.run(pos, diam, 40, oracle.params(adherence=0.5))
    assert np.array_equal(on[-1], ref)
