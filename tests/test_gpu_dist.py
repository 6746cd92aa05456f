"""The distributed runtime of libbdm.so (bdm_init_dist / bdm_init_dist_local, DESIGN.md §7;
north_star: x-slabs, halo exchange and migration with NCCL send/recv) against the CPU oracle.

Only one GPU is available to the tests, so the multi-rank data plane runs as virtual ranks
(bdm_init_dist_local): G ranks in one process over a 1-rank NCCL communicator, every message a
self send/recv -- the same kernels, protocol, fixed-capacity messages and device counts as G
processes.  Positions and displacements must equal oracle.run's bit for bit (ghosts keep their
global ids and canonical in-box order)."""
import os

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

    b.load_library()
    return b


def split_counts(n, G, rng):
    """An arbitrary initial distribution: random counts, agents in id order (not by slab)."""
    cuts = np.sort(rng.choice(np.arange(1, n), G - 1, replace=False)) if G > 1 else np.array([], int)
    return np.diff(np.concatenate([[0], cuts, [n]]))


def gather(bdm, h, what, n):
    ids, vals = bdm.bdm_get_local(h, what)
    ids, vals = to_np(ids), to_np(vals)
    out = np.full((n, 3), np.nan)
    seen = np.zeros(n, int)
    np.add.at(seen, ids, 1)
    out[ids] = vals
    assert np.all(seen == 1), "agents lost or duplicated"
    return out


def run_dist(bdm, pos, diam, G, steps, seed=0, device=True, stream=None, **kw):
    import torch

    n = len(diam)
    counts = split_counts(n, G, np.random.default_rng(seed))
    ids = np.arange(n, dtype=np.int64)
    prm = bdm.bdm_params_default(device=0, **kw)
    if device:
        h = bdm.bdm_init_dist_local(G, counts, torch.from_numpy(ids).cuda(), torch.from_numpy(pos).cuda(),
                                    torch.from_numpy(diam).cuda(), prm, stream=stream)
    else:
        h = bdm.bdm_init_dist_local(G, counts, ids, pos, diam, prm, stream=stream)
    bdm.bdm_mech_step(h, steps)
    p = gather(bdm, h, bdm.BDM_OWNED_POSITIONS, n)
    d = gather(bdm, h, bdm.BDM_LAST_DISPLACEMENTS, n)
    if device:
        torch.cuda.synchronize()
    return h, p, d


def to_np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else a


@pytest.mark.parametrize("G", [1, 2, 4, 7])
def test_dist_virtual_ranks_equal_oracle(bdm, G):
    """cfg2 window (40^3 lattice), 5 steps: the C-ABI distributed path equals oracle.run."""
    pos, diam = bdm_inputs.make_config(2, n=40 ** 3)
    h, p, d = run_dist(bdm, pos, diam, G, 5)
    o_p, o_dp = oracle.run(pos, diam, 5)
    assert np.array_equal(p, o_p) and np.array_equal(d, o_dp)
    st = bdm.bdm_get_stats(h)
    assert st["world"] == G and st["steps"] == 5 and st["n_agents"] == len(diam)
    if G > 1:
        assert st["migrated"] > 0 and st["ghosts"] > 0
        cuts = bdm.bdm_get_cuts(h)
        assert cuts[0] == -(2 ** 31) and cuts[-1] == 2 ** 31 - 1 and all(a < b for a, b in zip(cuts, cuts[1:]))


def test_dist_gaussian_host_inputs_across_chunks(bdm):
    """Gaussian cfg3 subset (work-balanced cuts differ from count cuts), host input arrays, 20 steps
    = two chunks (one host round trip each): equals oracle.run; the steps inside a chunk issue no
    host synchronisation (bdm_get_stats.host_syncs grows by exactly 1 per chunk)."""
    pos, diam = bdm_inputs.make_config(3, n=200_000)
    n = len(diam)
    counts = split_counts(n, 3, np.random.default_rng(4))
    h = bdm.bdm_init_dist_local(3, counts, np.arange(n, dtype=np.int64), pos, diam)
    s0 = bdm.bdm_get_stats(h)
    bdm.bdm_mech_step(h, 20)
    s1 = bdm.bdm_get_stats(h)
    assert s1["chunks"] - s0["chunks"] == 2 and s1["host_syncs"] - s0["host_syncs"] == 2
    p = gather(bdm, h, bdm.BDM_OWNED_POSITIONS, n)
    d = gather(bdm, h, bdm.BDM_LAST_DISPLACEMENTS, n)
    o_p, o_dp = oracle.run(pos, diam, 20)
    assert np.array_equal(p, o_p) and np.array_equal(d, o_dp)


def test_dist_overflow_rerun_is_exact(bdm, monkeypatch):
    """Messages of 16 records overflow at once: the chunk is re-run from its device checkpoint with
    larger buffers (stats.redo_chunks > 0) and the result is still oracle.run's."""
    monkeypatch.setenv("BDM_DIST_CAP0", "16")
    # (the variable is read at init)
    pos, diam = bdm_inputs.make_config(2, n=30 ** 3)
    h, p, d = run_dist(bdm, pos, diam, 4, 6, seed=2)
    assert bdm.bdm_get_stats(h)["redo_chunks"] > 0
    o_p, o_dp = oracle.run(pos, diam, 6)
    assert np.array_equal(p, o_p) and np.array_equal(d, o_dp)


def test_dist_small_diameters_single_rank_path(bdm):
    """Empty ranks and a rank count larger than the occupied layers do not break the protocol."""
    rng = np.random.default_rng(3)
    pos = rng.uniform(0.0, 40.0, (2000, 3))
    diam = rng.uniform(8.0, 12.0, 2000)
    h, p, d = run_dist(bdm, pos, diam, 8, 3, seed=5)
    o_p, o_dp = oracle.run(pos, diam, 3)
    assert np.array_equal(p, o_p) and np.array_equal(d, o_dp)


def test_dist_real_communicator_one_rank(bdm):
    """bdm_nccl_unique_id + bdm_init_dist with a real 1-rank NCCL communicator (the path bench.py's
    ranks take): equals oracle.run."""
    import torch

    pos, diam = bdm_inputs.make_config(1)
    n = len(diam)
    uid = bdm.bdm_nccl_unique_id()
    assert len(uid) == 128
    h = bdm.bdm_init_dist(torch.arange(n, dtype=torch.int64, device="cuda"), torch.from_numpy(pos).cuda(),
                          torch.from_numpy(diam).cuda(), rank=0, world=1, uid=uid, device=0)
    bdm.bdm_mech_step(h, 3)
    p = gather(bdm, h, bdm.BDM_OWNED_POSITIONS, n)
    o_p, _ = oracle.run(pos, diam, 3)
    assert np.array_equal(p, o_p)


def test_dist_rejects_bad_input(bdm):
    pos = np.zeros((3, 3))
    pos[1, 0] = np.nan
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_init_dist_local(2, [2, 1], np.arange(3, dtype=np.int64), pos, np.full(3, 10.0))
    assert e.value.code == bdm.BDM_EINVAL


def test_pair_digest_matches_oracle(bdm):
    """bdm_get_pair_digest (product handle, no BDM_RECORD) equals the oracle's per-agent neighbour /
    contact counts and order-free hashes (SURVEY §8(c) digest)."""
    pos, diam = bdm_inputs.make_config(1)
    h = bdm.bdm_init(pos, diam)
    o = oracle.step(pos, diam)
    for kind, kc, kh in ((0, "n_nb", "nb_hash"), (1, "n_ct", "ct_hash")):
        c, hs = bdm.bdm_get_pair_digest(h, kind)
        assert np.array_equal(c.astype(np.int64), o[kc].astype(np.int64))
        assert np.array_equal(hs, o[kh])


def test_dist_requires_small_moves(bdm):
    """The boundary-layer exchange needs |dp| < L (max_disp < box edge): rejected otherwise."""
    rng = np.random.default_rng(8)
    pos = rng.uniform(0.0, 100.0, (500, 3))
    diam = rng.uniform(1.0, 2.0, 500)  # L = 2 < max_disp = 3
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_init_dist_local(2, [250, 250], np.arange(500, dtype=np.int64), pos, diam)
    assert e.value.code == bdm.BDM_EINVAL and "max_disp" in str(e.value)


@pytest.mark.parametrize("G", [1, 3])
def test_dist_graph_replayed_steps_equal_oracle(bdm, G):
    """On a capturable stream the steady steps of a chunk are replayed as one CUDA graph per two steps
    (ThreadLocal stream capture, NCCL group included): 20 steps (two chunks, graph reused across
    them) equal oracle.run bit for bit."""
    import torch

    pos, diam = bdm_inputs.make_config(2, n=30 ** 3)
    st = torch.cuda.Stream()
    h, p, d = run_dist(bdm, pos, diam, G, 20, seed=6, stream=st)
    o_p, o_dp = oracle.run(pos, diam, 20)
    assert np.array_equal(p, o_p) and np.array_equal(d, o_dp)
    assert bdm.bdm_get_stats(h)["chunks"] == 2


def test_dist_new_batch_reuses_handle(bdm):
    """bdm_set_agents_dist: a second population through the same handle (communicator and buffers
    reused, cuts recomputed) is stepped exactly like a fresh one."""
    import torch

    st = torch.cuda.Stream()
    p1, d1 = bdm_inputs.make_config(2, n=25 ** 3)
    p2, d2 = bdm_inputs.random_instance(21, 9000, 260.0, 8.0, 12.0)
    uid = bdm.bdm_nccl_unique_id()
    h = bdm.bdm_init_dist(np.arange(len(d1), dtype=np.int64), p1, d1, rank=0, world=1, uid=uid, device=0, stream=st)
    bdm.bdm_mech_step(h, 3)
    bdm.bdm_set_agents_dist(h, np.arange(len(d2), dtype=np.int64), p2, d2)
    bdm.bdm_mech_step(h, 4)
    p = gather(bdm, h, bdm.BDM_OWNED_POSITIONS, len(d2))
    o_p, _ = oracle.run(p2, d2, 4)
    assert np.array_equal(p, o_p)


def test_dist_cuts_balance_work_not_count(bdm):
    """Gaussian population (dense core): the work-balanced cuts give the core ranks narrower slabs
    than count-balanced cuts would; every inner slab is at least 2 boxes wide."""
    pos, diam = bdm_inputs.make_config(3, n=400_000)
    n = len(diam)
    G = 4
    h = bdm.bdm_init_dist_local(G, [n // G] * (G - 1) + [n - (G - 1) * (n // G)], np.arange(n, dtype=np.int64),
                                pos, diam)
    cuts = bdm.bdm_get_cuts(h)
    L = float(diam.max())
    bx = np.floor(pos[:, 0] * (1.0 / (L * (1.0 + 2.0 ** -30)))).astype(np.int64)
    owned = [int(((bx >= cuts[g]) & (bx < cuts[g + 1])).sum()) for g in range(G)]
    assert all(b - a >= 2 for a, b in zip(cuts[1:-2], cuts[2:-1]))
    # the two central ranks hold fewer agents than the outer ones (their agents have more candidates)
    assert owned[1] < owned[0] and owned[2] < owned[3], owned
    ids, _ = bdm.bdm_get_local(h, bdm.BDM_OWNED_POSITIONS)
    assert len(ids) == n


def test_dist_handle_rejects_single_handle_calls(bdm):
    """Single-handle getters and setters on a distributed handle fail with ESTATE (no crash)."""
    pos, diam = bdm_inputs.make_config(1)
    h = bdm.bdm_init_dist_local(2, [2048, 2048], np.arange(4096, dtype=np.int64), pos, diam)
    for call in (lambda: bdm.bdm_grid_build(h), lambda: bdm.bdm_get_positions(h),
                 lambda: bdm.bdm_get_pairs(h, bdm.BDM_CONTACT), lambda: bdm.bdm_set_force_path(h, 1)):
        with pytest.raises(bdm.BdmError) as e:
            call()
        assert e.value.code == bdm.BDM_ESTATE
    bdm.bdm_mech_step(h, 1)
    assert len(bdm.bdm_get_local(h, bdm.BDM_LAST_DISPLACEMENTS)[0]) == 4096
