"""CPU tests of the x-slab protocol (paper_2006_06775_b200/dist.py), no GPU.

* LoopComm with G slabs in one process;
* world_size-2 torch.distributed over gloo (127.0.0.1), one slab per process;
both with the oracle-backed test engine (tests/slab_cpu_engine.py).  After K steps the gathered
positions must equal the single-process oracle trajectory bit for bit (north_star: halo exchange +
migration must not change any agent's neighbourhood)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bdm_inputs
import oracle
import slab_protocol as bdist
from slab_cpu_engine import CpuSlabEngine


def population(n=1500, seed=4):
    # elongated in x so that slabs are several boxes wide and agents cross cuts
    pos, diam = bdm_inputs.random_instance(seed, n, 1.0, 6.0, 14.0)
    rng = np.random.default_rng(seed)
    pos = np.stack([rng.uniform(0, 260, n), rng.uniform(0, 70, n), rng.uniform(0, 70, n)], axis=1)
    return pos, diam


def test_choose_bounds():
    hist = np.array([5, 5, 5, 5, 5, 5, 5, 5])
    b = bdist.choose_bounds(hist, 10, 4)
    assert b[0] == bdist.INT32_MIN and b[-1] == bdist.INT32_MAX
    assert b[1:-1] == [12, 14, 16]
    b = bdist.choose_bounds(np.array([100, 0, 0, 1]), 0, 3)  # every slab at least one box wide
    assert b[1:-1] == [1, 2]
    b = bdist.choose_bounds(np.array([7]), 3, 4)  # more slabs than boxes: strictly increasing
    assert all(x < y for x, y in zip(b, b[1:]))
    # enough boxes: inner slabs at least 2 wide (single-sync protocol), even for a spike
    b = bdist.choose_bounds(np.array([0, 0, 1000, 0, 0, 0, 0, 0, 0, 1]), 0, 4)
    assert all(y - x >= 2 for x, y in zip(b[1:-1], b[2:-1])), b


def _slab_work(b, bx, w, x0):
    cuts = [x0 - 1] + list(b[1:-1]) + [int(bx.max()) + 1]
    return np.array([w[max(a - x0, 0):c - x0].sum() for a, c in zip(cuts, cuts[1:])])


def test_work_weighted_bounds_balance_a_spheroid():
    """count-balanced cuts leave the core slabs of the Gaussian spheroid with more
    candidate work; cuts by estimated work (layer_work) balance it better, and a uniform population
    keeps count-like cuts."""
    rng = np.random.default_rng(3)
    n = 400_000
    sig = 992.2 * (n / 2e7) ** (1 / 3)
    pos = rng.normal(0.0, sig, (n, 3))
    diam = np.clip(np.exp(np.log(10.0) + 0.15 * rng.standard_normal(n)), 6.0, 16.0)
    inv = 1.0 / (16.0 * (1.0 + 2.0 ** -30))
    bc, bx = bdist.initial_bounds(pos, diam, 4, weighted=False)
    bw, _ = bdist.initial_bounds(pos, diam, 4, weighted=True)
    x0 = int(bx.min())
    w = bdist.layer_work(pos, inv, x0, int(bx.max()) - x0 + 1)
    imb = lambda b: (lambda v: v.max() / v.mean())(_slab_work(b, bx, w, x0))
    assert imb(bw) < imb(bc)
    # uniform density: the work estimate is proportional to the count, the cuts barely move
    pos_u = rng.uniform(0, 400, (n, 3))
    bu_c, _ = bdist.initial_bounds(pos_u, diam, 4, weighted=False)
    bu_w, _ = bdist.initial_bounds(pos_u, diam, 4, weighted=True)
    assert max(abs(a - c) for a, c in zip(bu_c[1:-1], bu_w[1:-1])) <= 1


def test_narrow_slab_falls_back_to_legacy_protocol():
    """A one-box-wide inner slab: an emigrant could land in a third rank's ghost layer, so the driver
    uses the legacy protocol, which stays exact."""
    pos, diam = population()
    _, bx = bdist.initial_bounds(pos, diam, 3)
    mid = int(np.median(bx))
    bounds = [bdist.INT32_MIN, mid, mid + 1, bdist.INT32_MAX]
    engines = []
    for g in range(3):
        m = np.flatnonzero((bx >= bounds[g]) & (bx < bounds[g + 1]))
        engines.append(CpuSlabEngine(m, pos[m], diam[m]))
    drv = bdist.SlabDriver(engines, bdist.LoopComm(3), bounds)
    assert not drv.fused
    for _ in range(2):
        drv.step()
    ref, _ = oracle.run(pos, diam, 2)
    ids = np.concatenate([e.owned()[0] for e in engines])
    got = np.concatenate([e.owned()[1] for e in engines])
    out = np.empty_like(got)
    out[ids] = got
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_loop_slabs_match_single_process(G, fused):
    """Both protocols: the single-sync one (split / one count exchange / ghosts = neighbour's boundary
    stayers + own emigrants) and the legacy one (six exchanges per step)."""
    pos, diam = population()
    steps = 3
    ref, _ = oracle.run(pos, diam, steps)
    bounds, bx = bdist.initial_bounds(pos, diam, G)
    engines = []
    for g in range(G):
        m = np.flatnonzero((bx >= bounds[g]) & (bx < bounds[g + 1]))
        engines.append(CpuSlabEngine(m, pos[m], diam[m]))
    drv = bdist.SlabDriver(engines, bdist.LoopComm(G), bounds, fused=fused)
    assert drv.fused == fused
    for _ in range(steps):
        drv.step()
    if G > 1:
        assert drv.migrated > 0 and drv.ghosts > 0  # the protocol was exercised (counts of the local slabs)
    ids = np.concatenate([e.owned()[0] for e in engines])
    got = np.concatenate([e.owned()[1] for e in engines])
    assert np.array_equal(np.sort(ids), np.arange(len(diam)))  # agents conserved, none duplicated
    out = np.empty_like(got)
    out[ids] = got
    assert np.array_equal(out, ref)


def test_loop_slabs_settle_from_arbitrary_distribution():
    """Ranks may start with any subset (bdm_init_dist semantics): the setup migrates every agent to
    its owner before the first step."""
    pos, diam = population(900, 7)
    G = 4
    bounds, _ = bdist.initial_bounds(pos, diam, G)
    assign = np.random.default_rng(0).integers(0, G, len(diam))
    engines = [CpuSlabEngine(np.flatnonzero(assign == g), pos[assign == g], diam[assign == g]) for g in range(G)]
    drv = bdist.SlabDriver(engines, bdist.LoopComm(G), bounds)
    drv.step()
    ref, _ = oracle.run(pos, diam, 1)
    ids = np.concatenate([e.owned()[0] for e in engines])
    got = np.concatenate([e.owned()[1] for e in engines])
    out = np.empty_like(got)
    out[ids] = got
    assert np.array_equal(out, ref)


def _worker(rank, world, port, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pos, diam = population(1200, 11)
        bounds, bx = bdist.initial_bounds(pos, diam, world)
        m = np.flatnonzero((bx >= bounds[rank]) & (bx < bounds[rank + 1]))
        eng = CpuSlabEngine(m, pos[m], diam[m])
        drv = bdist.SlabDriver([eng], bdist.TorchComm(torch.device("cpu")), bounds)
        assert drv.fused
        for _ in range(steps):
            drv.step()
        ids, p = eng.owned()
        got = [None] * world
        dist.all_gather_object(got, (ids, p))
        if rank == 0:
            q.put(got)
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_single_process():
    world, steps = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pos, diam = population(1200, 11)
    ref, _ = oracle.run(pos, diam, steps)
    ids = np.concatenate([g[0] for g in got])
    vals = np.concatenate([g[1] for g in got])
    assert np.array_equal(np.sort(ids), np.arange(len(diam)))
    out = np.empty_like(vals)
    out[ids] = vals
    assert np.array_equal(out, ref)
    # both ranks really owned agents (the cut is inside the population)
    assert all(len(g[0]) > 100 for g in got)
