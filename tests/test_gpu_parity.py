"""GPU parity: libbdm.so (through the C ABI) against the CPU oracle, element by element.

Contract (BASELINE.json north_star):
  * box coordinates, neighbour set N and contact set C: bit-exact;
  * one-step fp64 displacements: |g - o| <= max(1e-9 |o|, 1e-12) per component (adherence
    ambiguity band: either branch accepted);
  * multi-step: teacher-forced per-step parity + invariants.
Because the kernels sum each agent's terms in the oracle's canonical order with the same
separately-rounded operations, displacements are also checked for bit equality
(test_bit_exact_*), a stronger property than the contract.
"""
import numpy as np
import pytest

import bdm_inputs
import oracle

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module")
def bdm():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2006_06775_b200 as b

    b.load_library()
    return b


def run_gpu(bdm, pos, diam, steps=1, record=True, pairs=False, **kw):
    prm = bdm.bdm_params_default(**kw)
    if record:
        prm.flags |= bdm.BDM_RECORD
    h = bdm.bdm_init(pos, diam, prm)
    bdm.bdm_grid_build(h)
    boxes = bdm.bdm_get_box_coords(h)
    info = bdm.bdm_get_grid_info(h)
    pr = [bdm.bdm_get_pairs(h, kind) for kind in (0, 1)] if pairs else None
    bdm.bdm_mech_step(h, steps)
    out = dict(h=h, boxes=boxes, info=info, pairs=pr, dp=bdm.bdm_get_displacements(h),
               pos_new=bdm.bdm_get_positions(h))
    if record:
        out.update(bdm.bdm_get_agent_stats(h))
    return out


def assert_dp_contract(g_dp, o_dp, o_force=None, s_abs=None, adherence=0.1):
    tol = np.maximum(1e-9 * np.abs(o_dp), 1e-12)
    ok = (np.abs(g_dp - o_dp) <= tol).all(axis=1)
    if o_force is not None:
        band = np.abs(np.linalg.norm(o_force, axis=1) - adherence) <= 64 * U * s_abs
        ok |= band
    bad = np.flatnonzero(~ok)
    assert bad.size == 0, f"{bad.size} agents out of tolerance, first {bad[:5]}: {g_dp[bad[:3]]} vs {o_dp[bad[:3]]}"


def compare_full(bdm, pos, diam, pairs=True, **kw):
    g = run_gpu(bdm, pos, diam, pairs=pairs, **kw)
    # the product kernel (fp32 candidate prefilter, no statistics) must give the recorded kernel's
    # displacements bit for bit: the prefilter never drops a contact
    fast = run_gpu(bdm, pos, diam, record=False, **kw)
    assert np.array_equal(fast["dp"], g["dp"])
    prm = oracle.params(**{k: v for k, v in kw.items() if k in oracle.DEFAULTS})
    o = oracle.step(pos, diam, prm)
    gp = oracle.grid_params(pos, diam, prm.box_edge_min)
    assert g["info"]["L"] == gp["L"] and g["info"]["inv"] == gp["inv"]
    assert g["info"]["lo"] == gp["lo"] and g["info"]["hi"] == gp["hi"]
    assert np.array_equal(g["boxes"], oracle.box_coords(pos, diam, prm.box_edge_min))
    for k in ("n_cand", "n_nb", "n_ct", "nb_hash", "ct_hash"):
        assert np.array_equal(g[k], o[k]), k
    assert_dp_contract(g["dp"], o["dp"], o["force"], o["s_abs"], prm.adherence)
    assert np.array_equal(g["branch"], o["branch"])
    if pairs:
        for kind in (0, 1):
            assert np.array_equal(g["pairs"][kind], oracle.pairs(pos, diam, kind, prm)), kind
    return g, o


def test_cfg1_full_parity(bdm):
    pos, diam = bdm_inputs.make_config(1)
    g, o = compare_full(bdm, pos, diam)
    assert np.array_equal(g["pos_new"], o["pos_new"])


def test_bit_exact_cfg1(bdm):
    pos, diam = bdm_inputs.make_config(1)
    g = run_gpu(bdm, pos, diam, record=False)
    o = oracle.step(pos, diam, record=False)
    assert np.array_equal(g["dp"], o["dp"])


@pytest.mark.parametrize("dt", [1.0, 0.1])
def test_cfg2_full_parity(bdm, dt):
    """configs[1]: 10^6 agents, every agent compared (dt=0.1 exercises the free branch)."""
    pos, diam = bdm_inputs.make_config(2)
    g, o = compare_full(bdm, pos, diam, pairs=(dt == 1.0), dt=dt)
    assert np.array_equal(g["dp"], o["dp"])


@pytest.mark.parametrize("inst", range(12))
def test_random_instances(bdm, inst):
    """Ragged sizes, varied density, wide diameter range, coincident centres."""
    rng = np.random.default_rng(77 + inst)
    n = int(rng.integers(1, 5000))
    side = float(rng.uniform(20.0, 300.0)) * (n / 1000.0) ** (1 / 3)
    pos, diam = bdm_inputs.random_instance(inst + 500, n, side, 4.0, 16.0)
    if n > 3 and inst % 3 == 0:
        pos[2] = pos[1]
    compare_full(bdm, pos, diam, box_edge_min=0.0 if inst % 4 else 20.0)


def test_single_box_and_negative_coordinates(bdm):
    """All agents in one box (box_edge_min larger than the cloud) and negative coordinates."""
    pos, diam = bdm_inputs.random_instance(9, 700, 30.0, 6.0, 10.0)
    pos -= 100.0
    compare_full(bdm, pos, diam, box_edge_min=500.0)


def test_lattice_exact_zero(bdm):
    g = np.arange(6) * 9.0
    pos = np.array([(x, y, z) for x in g for y in g for z in g])
    diam = np.full(len(pos), 10.0)
    r = run_gpu(bdm, pos, diam, max_disp=100.0)
    idx = np.rint(pos / 9.0).astype(int)
    interior = ((idx > 0) & (idx < 5)).all(axis=1)
    assert np.all(r["dp"][interior] == 0.0)
    o = oracle.step(pos, diam, oracle.params(max_disp=100.0))
    assert np.array_equal(r["dp"], o["dp"])


def test_two_spheres_and_coincident(bdm):
    r = run_gpu(bdm, np.array([[0.0, 0, 0], [9.0, 0, 0]]), np.array([10.0, 10.0]))
    o = oracle.step(np.array([[0.0, 0, 0], [9.0, 0, 0]]), np.array([10.0, 10.0]))
    assert np.array_equal(r["dp"], o["dp"])
    pos = np.array([[1.0, 2, 3], [1.0, 2, 3], [50.0, 0, 0]])
    r = run_gpu(bdm, pos, np.array([10.0, 10.0, 10.0]), max_disp=1000.0)
    assert r["dp"].tolist() == [[-80.0, 0, 0], [80.0, 0, 0], [0.0, 0, 0]]


def test_empty_and_single(bdm):
    h = bdm.bdm_init(np.zeros((0, 3)), np.zeros(0))
    bdm.bdm_mech_step(h, 3)
    assert bdm.bdm_get_displacements(h).shape == (0, 3)
    r = run_gpu(bdm, np.array([[5.0, -3.0, 2.0]]), np.array([10.0]))
    assert r["dp"].tolist() == [[0.0, 0.0, 0.0]] and r["n_cand"].tolist() == [0]


def test_zero_steps_is_noop(bdm):
    pos, diam = bdm_inputs.make_config(1)
    h = bdm.bdm_init(pos, diam)
    bdm.bdm_mech_step(h, 0)
    assert np.array_equal(bdm.bdm_get_positions(h), pos)
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_get_displacements(h)
    assert e.value.code == bdm.BDM_ESTATE


def test_error_codes(bdm):
    bad = np.array([[0.0, np.nan, 0.0]])
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_init(bad, np.array([10.0]))
    assert e.value.code == bdm.BDM_EINVAL
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_init(np.zeros((2, 3)), np.array([10.0, -1.0]))
    assert e.value.code == bdm.BDM_EINVAL and "1" in str(e.value)
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_init(np.zeros((1, 3)), np.array([1.0]), bdm.bdm_params_default(eta=0.0))
    assert e.value.code == bdm.BDM_EINVAL
    h = bdm.bdm_init(np.array([[2.0 ** 21, 0, 0]]), np.array([1.0]))
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_mech_step(h, 1)
    assert e.value.code == bdm.BDM_ERANGE
    pos, diam = bdm_inputs.make_config(1)
    h = bdm.bdm_init(pos, diam)
    lib = bdm.load_library()
    import ctypes

    cnt = ctypes.c_int64(0)
    out = np.zeros((4, 2), np.int64)
    rc = lib.bdm_get_pairs(h.raw, 0, ctypes.byref(cnt), ctypes.c_void_p(out.ctypes.data), 2)
    assert rc == bdm.BDM_ETRUNC and cnt.value > 2


def test_multistep_teacher_forced(bdm):
    """BASELINE.json: multi-step runs compared by per-step parity and invariants.  Each step of the
    GPU run is checked against the oracle stepped from the GPU's own state at that step."""
    pos, diam = bdm_inputs.make_config(2, n=30 ** 3)
    prm = bdm.bdm_params_default()
    h = bdm.bdm_init(pos, diam, prm)
    cur = pos
    for s in range(10):
        bdm.bdm_mech_step(h, 1)
        dp = bdm.bdm_get_displacements(h)
        nxt = bdm.bdm_get_positions(h)
        o = oracle.step(cur, diam)
        assert_dp_contract(dp, o["dp"], o["force"], o["s_abs"])
        assert np.array_equal(nxt, cur + dp)
        assert np.all(np.linalg.norm(dp, axis=1) <= 3.0 * (1 + 4 * U))
        cur = nxt
    # free-running divergence vs the oracle's own trajectory is reported, not gated
    p_o, _ = oracle.run(pos, diam, 10)
    print("free-running max |dp| divergence after 10 steps:", np.abs(p_o - cur).max())


def test_deterministic_rerun(bdm):
    pos, diam = bdm_inputs.make_config(2, n=40 ** 3)
    a = run_gpu(bdm, pos, diam, steps=5, record=False)
    b = run_gpu(bdm, pos, diam, steps=5, record=False)
    assert np.array_equal(a["pos_new"], b["pos_new"]) and np.array_equal(a["dp"], b["dp"])


def test_device_pointer_path(bdm):
    import torch

    pos, diam = bdm_inputs.make_config(1)
    tp = torch.from_numpy(pos).cuda()
    td = torch.from_numpy(diam).cuda()
    h = bdm.bdm_init(tp, td)
    bdm.bdm_mech_step(h, 2)
    dp = bdm.bdm_get_displacements(h)
    torch.cuda.synchronize()
    hh = bdm.bdm_init(pos, diam)
    bdm.bdm_mech_step(hh, 2)
    assert np.array_equal(dp.cpu().numpy(), bdm.bdm_get_displacements(hh))


def test_device_generator_matches_numpy(bdm):
    import torch

    n = 100_003
    lo, hi = bdm_inputs.box_of(4, 2 * 10 ** 8)
    pos = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    diam = torch.empty(n, dtype=torch.float64, device="cuda")
    bdm.bdm_generate_uniform(4, 12345, n, lo, hi, 8.0, 12.0, pos, diam)
    torch.cuda.synchronize()
    p_np, d_np = bdm_inputs.uniform_population(4, np.arange(12345, 12345 + n), lo, hi, 8.0, 12.0)
    assert np.array_equal(pos.cpu().numpy(), p_np) and np.array_equal(diam.cpu().numpy(), d_np)


def test_prefilter_boundary_contacts(bdm):
    """Adversarial case for the conservative fp32 filter: pairs of largest-diameter agents (r_j = L/2,
    so the contact bound equals s) just inside contact (d = s (1 - 2^-40)) and just outside, far from
    the origin where fp32 rounds positions to ~1e-3 um, in random directions."""
    rng = np.random.default_rng(5)
    m = 4000
    base = rng.uniform(-9000.0, 9000.0, size=(m, 3))
    base[:, 0] = np.where(np.arange(m) % 2, 9990.0, -9990.0) + rng.uniform(-5, 5, m)
    u = rng.normal(size=(m, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    D = 12.0
    s = D  # two agents of diameter D: s = r_i + r_j = D
    frac = np.where(np.arange(m) % 3 == 0, 1.0 + 2.0 ** -40, 1.0 - 2.0 ** -40)
    # pairs 40 um apart along y, z (> 2 D: pairs do not interact)
    base[:, 1] = (np.arange(m) % 60) * 40.0 - 9000.0
    base[:, 2] = (np.arange(m) // 60) * 40.0 + 8000.0
    pos = np.concatenate([base, base + u * (s * frac)[:, None]])
    # plus pairs straddling box corners / edges diagonally (exercise the box culling of the
    # product kernel: the partner sits in a corner or edge neighbour box)
    Lb = 1.0 / (D * (1.0 + 2.0 ** -30))
    k = 600
    corner = np.stack([np.full(k, 7000.0), (np.arange(k) % 30) * 48.0 + 100.0, (np.arange(k) // 30) * 48.0 + 100.0], 1)
    corner = np.floor(corner * Lb) / Lb + 1e-9  # just above a box corner
    dirs = np.array([[-1, -1, -1], [-1, -1, 0], [-1, 0, -1], [0, -1, -1], [-1, 1, -1], [-1, -1, 1]], float)
    dd = dirs[np.arange(k) % len(dirs)]
    dd /= np.linalg.norm(dd, axis=1)[:, None]
    partner = corner + dd * (s * (1.0 - 2.0 ** -40))
    pos = np.concatenate([pos, corner, partner])
    diam = np.full(len(pos), D)
    o = oracle.step(pos, diam, oracle.params(max_disp=100.0), record=True)
    assert (o["n_ct"] > 0).sum() > m  # most pairs are in contact
    g = run_gpu(bdm, pos, diam, record=False, max_disp=100.0)
    assert np.array_equal(g["dp"], o["dp"])


def test_agents_on_box_faces(bdm):
    """Agents placed on, just below and just above box faces on every axis (x * inv within 1e-12 of an
    integer, also far from the origin): box coordinates, pair sets and displacements equal the
    oracle's (pins the product kernels' box assignment from the fp32 copy, which defers such
    agents to their fp64 position)."""
    rng = np.random.default_rng(9)
    D = 10.0
    edge = D * (1.0 + 2.0 ** -30)
    k = rng.integers(-200, 200, size=(3000, 3)).astype(float)
    k[::2, 0] += 700.0  # half of them far from the origin along x (larger fp32 rounding)
    # relative offsets from exactly on a face to beyond the fp32 decision margin (|t| 2^-21 ~ 4.8e-7 |t|)
    off = rng.choice([-2e-6, -1e-6, -5e-7, -4e-7, -1e-9, -1e-12, 0.0, 1e-12, 1e-9, 4e-7, 5e-7, 1e-6, 2e-6],
                     size=(3000, 3))
    pos = k * edge + off * np.maximum(1.0, np.abs(k * edge))
    # a partner in contact across a face for each
    u = rng.normal(size=(3000, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    pos = np.concatenate([pos, pos + 9.0 * u])
    diam = np.full(len(pos), D)
    compare_full(bdm, pos, diam, pairs=True)


@pytest.mark.slow
def test_cfg3_full_size_sampled(bdm):
    """configs[2] at full size (2e7 agents) in the launch configuration bench.py times: every
    statistic and displacement of a sample of agents (random + the densest core) against the
    oracle computed one by one on the same input."""
    pos, diam = bdm_inputs.make_config(3)
    g = run_gpu(bdm, pos, diam)
    fast = run_gpu(bdm, pos, diam, record=False)
    assert np.array_equal(fast["dp"], g["dp"])  # product kernel == recorded kernel, all 2e7 agents
    rng = np.random.default_rng(0)
    core = np.flatnonzero(np.linalg.norm(pos, axis=1) < 60.0)[:3000]
    sample = np.unique(np.concatenate([rng.choice(len(diam), 20000, replace=False), core]))
    o = oracle.step(pos, diam, sample=sample)
    for k in ("n_cand", "n_nb", "n_ct", "nb_hash", "ct_hash", "branch"):
        assert np.array_equal(g[k][sample], o[k][sample]), k
    assert_dp_contract(g["dp"][sample], o["dp"], o["force"][sample], o["s_abs"][sample])
    assert np.array_equal(g["dp"][sample], o["dp"])
    # whole-population properties: every agent's box is its floor(p*inv), |dp| <= max_disp
    assert np.array_equal(g["boxes"], np.floor(pos * g["info"]["inv"]).astype(np.int32))
    assert np.all(np.linalg.norm(g["dp"], axis=1) <= 3.0 * (1 + 4 * U))


@pytest.mark.slow
def test_cfg3_full_size_every_agent(bdm):
    """configs[2] at full size (2e7 agents), the bench's headline workload on the default product path:
    the displacements and new positions of EVERY agent equal one full oracle step bit for bit."""
    pos, diam = bdm_inputs.make_config(3)
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default())
    bdm.bdm_mech_step(h, 1)
    assert bdm.bdm_get_path_stats(h)["half"] == 1
    dp, p1 = bdm.bdm_get_displacements(h), bdm.bdm_get_positions(h)
    h.close()
    o = oracle.step(pos, diam, record=False)
    assert np.array_equal(dp, o["dp"])
    assert np.array_equal(p1, o["pos_new"])


@pytest.mark.slow
def test_cfg4_full_size_window(bdm):
    """configs[3] at full size (2e8 agents, generated on the device by K0) in the launch
    configuration bench.py times: the displacements of every agent inside a window are checked
    against the oracle run on that window plus a margin of two box edges (the window's agents have
    their complete 27-box neighbourhood in the oracle's input), with the global box edge."""
    import torch

    n = bdm_inputs.CFG_N[4]
    lo, hi = bdm_inputs.box_of(4, n)
    pos = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    diam = torch.empty(n, dtype=torch.float64, device="cuda")
    bdm.bdm_generate_uniform(4, 0, n, lo, hi, 8.0, 12.0, pos, diam)
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default())
    bdm.bdm_mech_step(h, 1)
    dp = bdm.bdm_get_displacements(h)
    torch.cuda.synchronize()
    L = float(diam.max().item())
    c = np.array([4000.0, 1500.0, 1500.0])
    w, m = 60.0, 2.2 * L
    sel = torch.all((pos > torch.tensor(c - w - m, device="cuda")) & (pos < torch.tensor(c + w + m, device="cuda")),
                    dim=1)
    idx = torch.nonzero(sel).squeeze(1)
    ps, ds, dps = pos[idx].cpu().numpy(), diam[idx].cpu().numpy(), dp[idx].cpu().numpy()
    inner = np.all(np.abs(ps - c) < w, axis=1)
    o = oracle.step(ps, ds, oracle.params(box_edge_min=L), sample=np.flatnonzero(inner), record=False)
    assert inner.sum() > 100
    assert np.array_equal(dps[inner], o["dp"])
