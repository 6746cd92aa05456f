"""Virtual x-slabs on one GPU: G slab handles of libbdm.so in one process exchanging
through LoopComm run the exact multi-GPU protocol of dist.py (pack / exchange / step / migrate
kernels) and must reproduce the CPU oracle's trajectory (oracle.run, DESIGN.md §3 O8) and the
single-handle run bit for bit.  Real multi-GPU NCCL runs use the
same driver with TorchComm (bench.py under torchrun)."""
import numpy as np
import pytest

import bdm_inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch

    assert torch.cuda.is_available()
    import paper_2006_06775_b200 as bdm
    import slab_protocol as bdist

    return torch, bdm, bdist


def run_single(bdm, pos, diam, steps):
    h = bdm.bdm_init(pos, diam)
    bdm.bdm_mech_step(h, steps)
    return bdm.bdm_get_positions(h), bdm.bdm_get_displacements(h)


def run_slabs(torch, bdist, pos, diam, steps, G, assign=None):
    bounds, bx = bdist.initial_bounds(pos, diam, G)
    engines = []
    n = len(diam)
    for g in range(G):
        m = np.flatnonzero((bx >= bounds[g]) & (bx < bounds[g + 1])) if assign is None else np.flatnonzero(assign == g)
        engines.append(bdist.GpuSlabEngine(torch.from_numpy(m).cuda(), torch.from_numpy(pos[m].copy()).cuda(),
                                           torch.from_numpy(diam[m].copy()).cuda(), capacity=n + 16))
    drv = bdist.SlabDriver(engines, bdist.LoopComm(G), bounds)
    for s in range(steps):
        drv.step(want_dp=(s == steps - 1))
    torch.cuda.synchronize()
    out = np.full((n, 3), np.nan)
    dp = np.full((n, 3), np.nan)
    seen = np.zeros(n, int)
    for e in engines:
        ids, p = e.owned()
        out[ids] = p
        seen[ids] += 1
        i2, d = e.last_dp()
        dp[i2] = d
    assert np.all(seen == 1), "agents lost or duplicated"
    return out, dp, drv


@pytest.mark.parametrize("G", [2, 4, 7])
def test_virtual_slabs_bit_identical(mods, G):
    """The slab kernels (pack, split, mark-dead, unpack, slab step) against the oracle: positions
    after 5 steps and the last step's displacements equal oracle.run's bit for bit."""
    torch, bdm, bdist = mods
    pos, diam = bdm_inputs.make_config(2, n=40 ** 3)
    steps = 5
    o_p, o_dp = oracle.run(pos, diam, steps)
    p, dp, drv = run_slabs(torch, bdist, pos, diam, steps, G)
    assert drv.migrated > 0 and drv.ghosts > 0
    assert np.array_equal(p, o_p)
    assert np.array_equal(dp, o_dp)
    ref_p, ref_dp = run_single(bdm, pos, diam, steps)
    assert np.array_equal(p, ref_p) and np.array_equal(dp, ref_dp)


def test_virtual_slabs_gaussian_and_arbitrary_start(mods):
    """Gaussian cfg3 subset with an arbitrary initial owner per agent (settled first): oracle.run."""
    torch, bdm, bdist = mods
    pos, diam = bdm_inputs.make_config(3, n=200_000)
    assign = np.random.default_rng(1).integers(0, 3, len(diam))
    o_p, o_dp = oracle.run(pos, diam, 3)
    p, dp, _ = run_slabs(torch, bdist, pos, diam, 3, 3, assign=assign)
    assert np.array_equal(p, o_p) and np.array_equal(dp, o_dp)


def test_virtual_slabs_small_diameters_large_moves(mods):
    """Diameters below max_disp (L = 2.5 um < max_disp = 3 um, dt large: agents can move more than a
    box per step).  The single-sync protocol assumes |dp| < L, so the driver must fall back to the
    legacy protocol here; positions and displacements still equal oracle.run's."""
    torch, bdm, bdist = mods
    rng = np.random.default_rng(11)
    n = 6000
    pos = rng.uniform(0.0, 60.0, (n, 3))
    diam = rng.uniform(1.5, 2.5, n)
    steps = 3
    o_p, o_dp = oracle.run(pos, diam, steps)
    p, dp, drv = run_slabs(torch, bdist, pos, diam, steps, 3)
    assert not drv.fused
    assert np.array_equal(p, o_p) and np.array_equal(dp, o_dp)
