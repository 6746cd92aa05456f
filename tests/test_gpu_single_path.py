"""The single-pass force kernel k_force as a product path: it runs when selected per
handle with bdm_set_force_path(BDM_PATH_SINGLE), in RECORD / skip steps, and when neither the pair
rows nor a ring of them fit (the 10^9-agent single-GPU run now takes the banded ring phase, also
checked here at full size).  Checked against the CPU oracle element by element, like the
default path (BASELINE.json north_star parity contract), plus the ENONFINITE
diagnosis (a non-finite force aborts with the offending pair)."""
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


def single_step(bdm, pos, diam, steps=1, **kw):
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(**kw))
    bdm.bdm_set_force_path(h, bdm.BDM_PATH_SINGLE)
    bdm.bdm_mech_step(h, steps)
    assert bdm.bdm_get_path_stats(h)["half"] == 0  # k_force ran
    return bdm.bdm_get_displacements(h), bdm.bdm_get_positions(h)


@pytest.mark.parametrize("dt", [1.0, 0.1])
def test_single_pass_cfg2_full(bdm, dt):
    """configs[1] (10^6 agents), every agent: k_force's displacements equal the oracle's bit for bit
    (dt = 0.1 takes the free branch for ~12% of the agents)."""
    pos, diam = bdm_inputs.make_config(2)
    dp, p1 = single_step(bdm, pos, diam, dt=dt)
    o = oracle.step(pos, diam, oracle.params(dt=dt), record=False)
    assert np.array_equal(dp, o["dp"])
    assert np.array_equal(p1, o["pos_new"])


def test_single_pass_cfg1_multistep(bdm):
    """Five steps of k_force equal five oracle steps (the oracle's own trajectory, bit for bit)."""
    pos, diam = bdm_inputs.make_config(1)
    _, p = single_step(bdm, pos, diam, steps=5)
    po, _ = oracle.run(pos, diam, 5)
    assert np.array_equal(p, po)


def test_single_pass_prefilter_adversarial(bdm):
    """The fp32 prefilter and box culling of k_force on the adversarial near-contact pairs far from
    the origin (d = s (1 -+ 2^-40)) and across box corners (see test_gpu_parity)."""
    rng = np.random.default_rng(5)
    m, D = 4000, 12.0
    base = rng.uniform(-9000.0, 9000.0, size=(m, 3))
    base[:, 0] = np.where(np.arange(m) % 2, 9990.0, -9990.0) + rng.uniform(-5, 5, m)
    base[:, 1] = (np.arange(m) % 60) * 40.0 - 9000.0
    base[:, 2] = (np.arange(m) // 60) * 40.0 + 8000.0
    u = rng.normal(size=(m, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    frac = np.where(np.arange(m) % 3 == 0, 1.0 + 2.0 ** -40, 1.0 - 2.0 ** -40)
    pos = np.concatenate([base, base + u * (D * frac)[:, None]])
    Lb = 1.0 / (D * (1.0 + 2.0 ** -30))
    k = 600
    corner = np.stack([np.full(k, 7000.0), (np.arange(k) % 30) * 48.0 + 100.0, (np.arange(k) // 30) * 48.0 + 100.0], 1)
    corner = np.floor(corner * Lb) / Lb + 1e-9
    dirs = np.array([[-1, -1, -1], [-1, -1, 0], [-1, 0, -1], [0, -1, -1], [-1, 1, -1], [-1, -1, 1]], float)
    dd = dirs[np.arange(k) % len(dirs)]
    dd /= np.linalg.norm(dd, axis=1)[:, None]
    pos = np.concatenate([pos, corner, corner + dd * (D * (1.0 - 2.0 ** -40))])
    diam = np.full(len(pos), D)
    o = oracle.step(pos, diam, oracle.params(max_disp=100.0), record=False)
    dp, _ = single_step(bdm, pos, diam, max_disp=100.0)
    assert np.array_equal(dp, o["dp"])


def test_single_pass_box_faces(bdm):
    """Agents on, just below and just above box faces (relative offsets 0 .. 2e-6), far from the
    origin too, each with a contact partner across the face."""
    rng = np.random.default_rng(9)
    D = 10.0
    edge = D * (1.0 + 2.0 ** -30)
    k = rng.integers(-200, 200, size=(3000, 3)).astype(float)
    k[::2, 0] += 700.0
    off = rng.choice([-2e-6, -1e-6, -5e-7, -4e-7, -1e-9, -1e-12, 0.0, 1e-12, 1e-9, 4e-7, 5e-7, 1e-6, 2e-6],
                     size=(3000, 3))
    pos = k * edge + off * np.maximum(1.0, np.abs(k * edge))
    u = rng.normal(size=(3000, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    pos = np.concatenate([pos, pos + 9.0 * u])
    diam = np.full(len(pos), D)
    dp, _ = single_step(bdm, pos, diam)
    assert np.array_equal(dp, oracle.step(pos, diam, record=False)["dp"])


def test_force_path_switch_rejects_bad_value(bdm):
    h = bdm.bdm_init(np.zeros((1, 3)), np.array([1.0]))
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_set_force_path(h, 7)
    assert e.value.code == bdm.BDM_EINVAL


def test_nonfinite_force_names_the_pair(bdm):
    """"abort with a diagnostic naming the offending pair".  k = 1e308 (finite, valid)
    makes k * delta overflow for the overlapping pair (3, 7); the other agents are far apart.  Both
    force paths report BDM_ENONFINITE with the pair."""
    pos = np.array([[100.0 * i, 0.0, 0.0] for i in range(10)])
    pos[7] = pos[3] + np.array([5.0, 0.0, 0.0])
    diam = np.full(10, 10.0)
    for path in (bdm.BDM_PATH_AUTO, bdm.BDM_PATH_SINGLE):
        h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(k_rep=1e308))
        bdm.bdm_set_force_path(h, path)
        with pytest.raises(bdm.BdmError) as e:
            bdm.bdm_mech_step(h, 1)
            bdm.bdm_sync(h)
        assert e.value.code == bdm.BDM_ENONFINITE
        assert "(3, 7)" in str(e.value), str(e.value)


def cfg5_window_step(bdm, path):
    """configs[4] at full size: 10^9 agents generated on the device (K0) on ONE GPU, one step on the
    given force path; returns the path taken and (window agents' displacements, oracle's)."""
    import torch

    n = bdm_inputs.CFG_N[5]
    lo, hi = bdm_inputs.box_of(5, n)
    free, _ = torch.cuda.mem_get_info()
    if free < 170e9:
        pytest.skip(f"needs ~170 GB of free device memory, {free / 1e9:.0f} GB free")
    pos = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    diam = torch.empty(n, dtype=torch.float64, device="cuda")
    bdm.bdm_generate_uniform(5, 0, n, lo, hi, 8.0, 12.0, pos, diam)
    torch.cuda.synchronize()
    L = float(diam.max().item())
    c = np.array([5000.0, 5000.0, 5000.0])
    w, m = 50.0, 2.2 * L
    idx = []
    step = 50_000_000
    for a in range(0, n, step):  # window selection in chunks (bounded temporaries)
        p = pos[a:a + step]
        sel = torch.all((p > torch.tensor(c - w - m, device="cuda")) & (p < torch.tensor(c + w + m, device="cuda")),
                        dim=1)
        idx.append(torch.nonzero(sel).squeeze(1) + a)
    idx = torch.cat(idx)
    ps, ds = pos[idx].cpu().numpy(), diam[idx].cpu().numpy()
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default())
    del pos, diam, p, sel
    torch.cuda.empty_cache()
    bdm.bdm_set_force_path(h, path)
    bdm.bdm_mech_step(h, 1)
    taken = bdm.bdm_get_path_stats(h)["half"]
    dp = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    bdm.bdm_get_displacements(h, dp)
    dps = dp[idx].cpu().numpy()
    del dp
    h.close()
    torch.cuda.empty_cache()
    inner = np.all(np.abs(ps - c) < w, axis=1)
    assert inner.sum() > 100
    o = oracle.step(ps, ds, oracle.params(box_edge_min=L), sample=np.flatnonzero(inner), record=False)
    return taken, dps[inner], o["dp"]


@pytest.mark.slow
def test_cfg5_full_size_window_single_pass(bdm):
    """configs[4] at full size on one GPU with the single-pass k_force (BDM_PATH_SINGLE): every agent of
    a window is checked against the oracle run on the window plus a margin of 2.2 box edges, with the
    global box edge."""
    taken, dp, odp = cfg5_window_step(bdm, bdm.BDM_PATH_SINGLE)
    assert taken == 0
    assert np.array_equal(dp, odp)


@pytest.mark.slow
def test_cfg5_full_size_window_ring(bdm):
    """configs[4] at full size on one GPU with the default path: the pair rows of 10^9 agents do not fit
    beside the state, so the half-shell phase runs band by band over a ring of rows (path 2, the launch
    configuration DESIGN.md §6.5 measures); the window check as above."""
    taken, dp, odp = cfg5_window_step(bdm, bdm.BDM_PATH_AUTO)
    assert taken == 2
    assert np.array_equal(dp, odp)
