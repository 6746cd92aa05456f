"""Half-shell pair path (k_half_search + k_half_sum) against the CPU oracle.

The plain product step tests each candidate pair once (forward half of the 27 boxes) and sums every
agent's contacts in canonical order from its backward/forward pair rows.  These tests pin:
  * bit equality with the oracle (and with the single-pass RECORD kernel) on ordinary inputs;
  * populations built so that pair rows overflow (a large sphere with ~48 small partners, placed
    near the upper corner of its box -> ~42 forward partners; near the lower corner -> ~42
    backward partners): those agents take the exact full-search path, results unchanged;
  * multi-step trajectories through the overflow path, bit-equal to the oracle's.
"""
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


def fib_sphere(n, r, c):
    k = np.arange(n) + 0.5
    phi = np.arccos(1.0 - 2.0 * k / n)
    th = np.pi * (1.0 + 5.0 ** 0.5) * k
    u = np.stack([np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi), np.cos(phi)], axis=1)
    return c + r * u


def hub_population(seed, n_bg=3000, partners=48):
    """Background agents plus hubs (D = 16, the box edge) each carrying `partners` small (D = 6)
    agents at distance 9.5 (all in contact with the hub, overlapping each other).  Hub ids come
    before their partners'.  Corners: 'hi' -> most partners follow the hub in sorted order (forward
    row overflow), 'lo' -> most precede it (backward row overflow)."""
    rng = np.random.default_rng(seed)
    L = 16.0
    pos = [rng.uniform(0.0, 240.0, (n_bg, 3))]
    diam = [rng.uniform(6.0, 12.0, n_bg)]
    for corner, box in (("hi", (3, 3, 3)), ("lo", (9, 4, 6)), ("hi", (6, 10, 2)), ("lo", (12, 12, 12))):
        off = 15.5 if corner == "hi" else 0.5
        c = np.array(box, float) * L + off
        pos.append(c[None, :])
        diam.append(np.array([16.0]))
        pos.append(fib_sphere(partners, 9.5, c))
        diam.append(np.full(partners, 6.0))
    return np.concatenate(pos), np.concatenate(diam)


def run(bdm, pos, diam, steps=1, record=False):
    prm = bdm.bdm_params_default()
    if record:
        prm.flags |= bdm.BDM_RECORD
    h = bdm.bdm_init(pos, diam, prm)
    bdm.bdm_mech_step(h, steps)
    return h, bdm.bdm_get_displacements(h), bdm.bdm_get_positions(h), bdm.bdm_get_path_stats(h)


def test_half_path_used_and_bit_exact_cfg1(bdm):
    pos, diam = bdm_inputs.make_config(1)
    h, dp, _, st = run(bdm, pos, diam)
    assert st["half"] == 1 and st["slow"] == 0
    _, dp_rec, _, st_rec = run(bdm, pos, diam, record=True)
    assert st_rec["half"] == 0  # statistics need the single-pass kernel
    assert np.array_equal(dp, dp_rec)
    assert np.array_equal(dp, oracle.step(pos, diam)["dp"])


@pytest.mark.parametrize("seed", [0, 1])
def test_row_overflow_takes_exact_path(bdm, seed):
    pos, diam = hub_population(seed)
    h, dp, _, st = run(bdm, pos, diam)
    assert st["half"] == 1
    assert st["slow"] >= 4, st  # the four hubs at least (their rows cannot hold ~42 partners)
    o = oracle.step(pos, diam)
    assert (o["n_ct"] > 32).sum() >= 4
    assert np.array_equal(dp, o["dp"])
    _, dp_rec, _, _ = run(bdm, pos, diam, record=True)
    assert np.array_equal(dp, dp_rec)


def test_row_overflow_multistep_trajectory(bdm):
    pos, diam = hub_population(7, n_bg=1500)
    _, _, p_gpu, _ = run(bdm, pos, diam, steps=4)
    p_orc, _ = oracle.run(pos, diam, 4)
    assert np.array_equal(p_gpu, p_orc)


def test_dense_random_cluster_bit_exact(bdm):
    """A jammed cluster at 3x lattice density: many agents with 20-40 contacts (rows overflow
    sporadically), bit-equal to the oracle."""
    rng = np.random.default_rng(11)
    n = 6000
    side = (n / 3.0e-3) ** (1.0 / 3.0)
    pos = rng.uniform(-side / 2, side / 2, (n, 3))
    diam = np.clip(np.exp(np.log(10.0) + 0.15 * rng.standard_normal(n)), 6.0, 16.0)
    _, dp, _, st = run(bdm, pos, diam)
    assert st["half"] == 1
    assert np.array_equal(dp, oracle.step(pos, diam)["dp"])
