"""Pins for the CPU oracle (run with -m "not gpu").

The oracle (oracle/bdm_oracle.c, grid) is checked against things other than itself:
closed forms of the force law (tests/golden/closed_forms.json), SPEC.md's worked examples
(tests/golden/spec_examples.json), exact invariants (lattice cancellation, Newton's third law,
rotation by 90 degrees), the independent O(N^2) brute force (oracle/brute.py), and an energy
descent property of the overdamped flow.  Each test names the passage it follows.
"""
import json
import math
import os

import numpy as np
import pytest

import bdm_inputs
from oracle import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def ulps(a, b):
    a, b = float(a), float(b)
    if a == b:
        return 0.0
    return abs(a - b) / (math.ulp(max(abs(a), abs(b))))


# ---------------------------------------------------------------- closed forms (north_star force law)
def test_two_sphere_closed_forms(orc):
    g = gold("closed_forms.json")["equal_spheres_D10"]
    for c in g["cases"]:
        hit, t = orc.pair_force([0.0, 0.0, 0.0], [c["d"], 0.0, 0.0], 10.0, 10.0)
        f = float(c["f"])
        if c["delta"] <= 0:
            assert not hit and np.all(t == 0.0), c
            continue
        assert hit
        # force on i (at origin) is f * (p_i - p_j)/d = -f x_hat: repulsive pushes i to -x
        assert ulps(-t[0], f) <= 2, (c, t)
        assert t[1] == 0.0 and t[2] == 0.0


def test_force_minimum_and_attraction_window(orc):
    # f(delta) = k delta - gamma sqrt(r delta): minimum -gamma^2 r/(4k) = -1 at delta = 0.1 (r = 2.5)
    hit, t = orc.pair_force([0.0, 0.0, 0.0], [9.9, 0.0, 0.0], 10.0, 10.0)
    assert hit and abs(t[0] - (-1.0) * -1.0) < 1e-12  # force on i is -f x_hat, f = -1
    for d, attractive in ((9.7, True), (9.65, True), (9.55, False), (9.3, False), (9.95, True)):
        hit, t = orc.pair_force([0.0, 0.0, 0.0], [d, 0.0, 0.0], 10.0, 10.0)
        # attraction (f < 0) iff delta < gamma^2 r / k^2 = 0.4  ->  force on i points +x
        assert hit and ((t[0] > 0) == attractive), (d, t)


def test_unequal_radii_direction(orc):
    g = gold("closed_forms.json")["unequal_spheres"]
    hit, t = orc.pair_force([0.0, 0.0, 0.0], [4.5, 6.0, 0.0], 4.0, 12.0)
    f = float(g["f"])
    assert hit
    assert abs(t[0] - f * -0.6) <= 4 * U * f and abs(t[1] - f * -0.8) <= 4 * U * f and t[2] == 0.0
    # swapping the operands negates the force bit-exactly (Newton's third law)
    hit2, t2 = orc.pair_force([4.5, 6.0, 0.0], [0.0, 0.0, 0.0], 12.0, 4.0)
    assert hit2 and np.array_equal(t2, -t)


def test_coincident_centres(orc):
    hit, t_hi = orc.pair_force([1.0, 2.0, 3.0], [1.0, 2.0, 3.0], 10.0, 10.0, idi=7, idj=3)
    assert hit and t_hi.tolist() == [80.0, 0.0, 0.0]
    hit, t_lo = orc.pair_force([1.0, 2.0, 3.0], [1.0, 2.0, 3.0], 10.0, 10.0, idi=3, idj=7)
    assert hit and t_lo.tolist() == [-80.0, 0.0, 0.0]


# ---------------------------------------------------------------- displacement rule (O6)
def test_two_sphere_displacement_clamp_and_free(orc):
    pos = np.array([[0.0, 0.0, 0.0], [9.0, 0.0, 0.0]])
    diam = np.array([10.0, 10.0])
    r = orc.step(pos, diam)
    # |F| = 3.675 > max_disp = 3 at dt = 1 -> clamped to 3 along the line of centres
    assert ulps(r["dp"][0, 0], -3.0) <= 2 and ulps(r["dp"][1, 0], 3.0) <= 2
    assert np.all(r["dp"][:, 1:] == 0.0)
    assert r["branch"].tolist() == [1, 1]
    r = orc.step(pos, diam, orc.params(dt=0.1))
    f = float(gold("closed_forms.json")["equal_spheres_D10"]["cases"][0]["f"])
    assert ulps(r["dp"][0, 0], -0.1 * f) <= 2 and ulps(r["dp"][1, 0], 0.1 * f) <= 2
    assert r["branch"].tolist() == [2, 2]


def test_adherence_threshold(orc):
    # D=4 spheres 3.75 apart: delta = 0.25, r = 1, f = 10*0.25 - gamma*0.5
    pos = np.array([[0.0, 0.0, 0.0], [3.75, 0.0, 0.0]])
    diam = np.array([4.0, 4.0])
    r = orc.step(pos, diam, orc.params(gamma_att=4.9))  # f = 0.05 <= 0.1 -> no motion
    assert np.all(r["dp"] == 0.0) and r["branch"].tolist() == [0, 0]
    r = orc.step(pos, diam, orc.params(gamma_att=4.7))  # f = 0.15 > 0.1 -> free move F*dt/eta
    assert r["branch"].tolist() == [2, 2]
    assert abs(r["dp"][0, 0] + 0.15) < 1e-12 and abs(r["dp"][1, 0] - 0.15) < 1e-12


def test_displacement_rule_direct(orc):
    dp, br = orc.displacement([0.06, 0.08, 0.0])  # |F| = 0.1 exactly at threshold -> no motion
    assert br == 0 and dp.tolist() == [0.0, 0.0, 0.0]
    dp, br = orc.displacement([30.0, 40.0, 0.0])  # |F| = 50, clamp to 3: (1.8, 2.4, 0)
    assert br == 1 and abs(dp[0] - 1.8) < 4e-16 and abs(dp[1] - 2.4) < 4e-16
    dp, br = orc.displacement([0.3, 0.4, 0.0], orc.params(dt=2.0, eta=4.0))  # c = 0.5 -> free
    assert br == 2 and dp.tolist() == [0.15, 0.2, 0.0]


@pytest.mark.parametrize("case", ["touching_zero_force"])
def test_spec_zero_force(orc, case):
    g = gold("spec_examples.json")[case]
    r = orc.step(np.array(g["pos"]), np.array(g["diam"]))
    assert np.array_equal(r["dp"], np.array(g["dp"]))


def test_separated_no_motion(orc):
    pos = np.array([[0.0, 0.0, 0.0], [11.0, 0.0, 0.0], [100.0, 0.0, 0.0]])
    r = orc.step(pos, np.array([10.0, 10.0, 10.0]))
    assert np.all(r["dp"] == 0.0) and np.all(r["n_ct"] == 0)


# ---------------------------------------------------------------- grid (O1-O3) against SPEC examples
def test_spec_rebuild_example(orc):
    g = gold("spec_examples.json")["rebuild_two_agents"]
    gp = orc.grid_params(np.array(g["pos"]), np.array(g["diam"]))
    assert gp["L"] == g["box_edge"]
    b = np.floor(np.array(g["pos"]) * gp["inv"]).astype(int)
    assert b.tolist() == g["boxes"]
    assert gp["lo"] == (0, 0, 0) and gp["hi"] == (2, 0, 0)


def test_spec_neighbour_examples(orc):
    ex = gold("spec_examples.json")
    for name in ("neighbours_within_r", "no_neighbours_beyond_r"):
        g = ex[name]
        prm = orc.params(box_edge_min=g.get("box_edge_min", 0.0))
        nb = orc.pairs(np.array(g["pos"]), np.array(g["diam"]), 0, prm)
        assert nb.tolist() == g["neighbour_pairs"], name


def test_negative_coordinates_floor(orc):
    pos = np.array([[-0.5, -10.5, 0.0], [0.5, 9.5, 0.0]])
    gp = orc.grid_params(pos, np.array([10.0, 10.0]))
    assert gp["lo"] == (-1, -2, 0) and gp["hi"] == (0, 0, 0)


def test_empty_and_single(orc):
    r = orc.step(np.zeros((0, 3)), np.zeros(0))
    assert r["dp"].shape == (0, 3)
    r = orc.step(np.array([[1.0, 2.0, 3.0]]), np.array([10.0]))
    assert np.all(r["dp"] == 0.0) and r["n_cand"][0] == 0


def test_invalid_inputs(orc):
    with pytest.raises(orc.OracleError):
        orc.step(np.array([[0.0, 0.0, np.nan]]), np.array([1.0]))
    with pytest.raises(orc.OracleError):
        orc.step(np.array([[0.0, 0.0, 0.0]]), np.array([0.0]))
    with pytest.raises(orc.OracleError):
        orc.step(np.array([[0.0, 0.0, 0.0]]), np.array([1.0]), orc.params(eta=0.0))
    with pytest.raises(orc.OracleError):  # |p*inv| >= 2^20 boxes breaks the 2^-30 margin (R9)
        orc.step(np.array([[2.0 ** 21, 0.0, 0.0]]), np.array([1.0]))


# ---------------------------------------------------------------- exact invariants
def lattice(side, s, D):
    g = np.arange(side) * s
    pos = np.array([(x, y, z) for x in g for y in g for z in g], dtype=np.float64)
    return pos, np.full(len(pos), D)


def test_lattice_cancellation(orc):
    """Simple-cubic lattice s=9, D=10: only axial pairs touch (9*sqrt2 > L=10).  Interior agents
    feel exactly zero force; faces f, edges sqrt2 f, corners sqrt3 f, pointing outward."""
    side = 5
    pos, diam = lattice(side, 9.0, 10.0)
    r = orc.step(pos, diam, orc.params(max_disp=100.0))
    F = r["force"]
    f = float(gold("closed_forms.json")["equal_spheres_D10"]["cases"][0]["f"])
    idx = np.rint(pos / 9.0).astype(int)
    boundary = ((idx == 0) | (idx == side - 1)).sum(axis=1)
    assert np.all(F[boundary == 0] == 0.0)
    for nb, mult in ((1, 1.0), (2, math.sqrt(2.0)), (3, math.sqrt(3.0))):
        mag = np.linalg.norm(F[boundary == nb], axis=1)
        assert np.all(np.abs(mag - mult * f) < 1e-13), nb
    # outward: sign of each nonzero component equals the side it sits on
    out = np.where(idx == 0, -1, np.where(idx == side - 1, 1, 0))
    assert np.array_equal(np.sign(F).astype(int), out)
    assert np.all(r["n_ct"] == (6 - boundary))


def test_symmetric_centroid(orc):
    """a sphere at the centroid of an equilateral triangle of equal spheres with equal
    overlaps feels no net force."""
    R = 8.0
    pos = [(R * math.cos(a), R * math.sin(a), 0.0) for a in (0.0, 2 * math.pi / 3, 4 * math.pi / 3)]
    pos = np.array(pos + [(0.0, 0.0, 0.0)])
    r = orc.step(pos, np.full(4, 10.0), orc.params(max_disp=100.0))
    assert np.linalg.norm(r["force"][3]) < 1e-13
    assert r["n_ct"][3] == 3


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_newton_third_law_sum(orc, seed):
    pos, diam = bdm_inputs.random_instance(seed, 1500, 90.0)
    r = orc.step(pos, diam)
    tot = r["force"].sum(axis=0)
    assert np.all(np.abs(tot) <= len(diam) * 4 * U * r["s_abs"].max())


def test_rotation_90_about_z(orc):
    """(x,y,z) -> (-y,x,z) maps every per-pair term bit-exactly; sums agree to summation order."""
    pos, diam = bdm_inputs.random_instance(5, 1200, 80.0)
    rot = np.stack([-pos[:, 1], pos[:, 0], pos[:, 2]], axis=1)
    a = orc.step(pos, diam, orc.params(max_disp=100.0))
    b = orc.step(rot, diam, orc.params(max_disp=100.0))
    assert np.array_equal(orc.pairs(pos, diam, 0), orc.pairs(rot, diam, 0))
    assert np.array_equal(orc.pairs(pos, diam, 1), orc.pairs(rot, diam, 1))
    Fa, Fb = a["force"], b["force"]
    want = np.stack([-Fa[:, 1], Fa[:, 0], Fa[:, 2]], axis=1)
    tol = 8 * U * a["s_abs"][:, None] + 1e-300
    assert np.all(np.abs(Fb - want) <= tol)
    assert np.array_equal(a["n_ct"], b["n_ct"]) and np.array_equal(a["nb_hash"], b["nb_hash"])


def energy(pos, diam, prm):
    nb, ct, _ = brute.all_pairs(pos, diam, prm)
    Uc = 0.0
    for i, j in ct:
        d = math.dist(pos[i], pos[j])
        ri, rj = diam[i] / 2, diam[j] / 2
        dl = ri + rj - d
        r = ri * rj / (ri + rj)
        Uc += prm["k_rep"] * dl * dl / 2 - (2.0 / 3.0) * prm["gamma_att"] * math.sqrt(r) * dl ** 1.5
    return Uc


def test_energy_descent_small_dt(orc):
    """dU/d(delta) = f, so the overdamped flow at small dt (no clamp) is a gradient descent of
    U = sum_C [k delta^2/2 - (2/3) gamma sqrt(r) delta^(3/2)] (SPEC.md:245 analogue)."""
    pos, diam = bdm_inputs.random_instance(11, 300, 45.0)
    kw = dict(dt=0.01, max_disp=100.0, adherence=0.0)
    prm = orc.params(**kw)
    e = [energy(pos, diam, dict(brute.DEFAULTS, **kw))]
    for _ in range(5):
        pos = orc.step(pos, diam, prm)["pos_new"]
        e.append(energy(pos, diam, dict(brute.DEFAULTS, **kw)))
    assert all(b <= a + 1e-9 for a, b in zip(e, e[1:])), e
    assert e[-1] < e[0]


# ---------------------------------------------------------------- grid oracle == brute force
DENSITIES = [40.0, 60.0, 90.0, 140.0, 250.0]


@pytest.mark.parametrize("inst", range(50))
def test_grid_equals_brute_force(orc, inst):
    """SPEC.md:665 acceptance #1 / SPEC.md:166: 50 randomized instances (<= 2000 agents, varied
    densities): grid neighbour and contact sets equal brute-force all-pairs sets exactly; per-pair
    terms identical; per-agent sums agree to summation order (the brute force sums by ascending id,
    the grid oracle in box order)."""
    rng = np.random.default_rng(1000 + inst)
    n = int(rng.integers(2, 400 if inst % 5 else 2000))
    side = DENSITIES[inst % 5] * (n / 400.0) ** (1.0 / 3.0)
    pos, diam = bdm_inputs.random_instance(inst, n, side, 6.0, 16.0 if inst % 3 == 0 else 12.0)
    if inst % 7 == 0:
        pos[1] = pos[0]  # coincident centres (R8)
    b = brute.step(pos, diam)
    g = orc.step(pos, diam)
    assert np.array_equal(orc.pairs(pos, diam, 0), b["nb"])
    assert np.array_equal(orc.pairs(pos, diam, 1), b["ct"])
    assert np.array_equal(g["n_nb"], b["n_nb"]) and np.array_equal(g["n_ct"], b["n_ct"])
    tol = np.maximum(1e-9 * np.abs(b["dp"]), 1e-12)
    band = np.abs(np.linalg.norm(b["force"], axis=1) - 0.1) <= 64 * U * b["s_abs"]
    ok = (np.abs(g["dp"] - b["dp"]) <= tol).all(axis=1) | band
    assert ok.all()
    assert np.array_equal(g["branch"][~band], b["branch"][~band])


def test_cfg1_grid_equals_brute_force(orc):
    pos, diam = bdm_inputs.make_config(1)
    b = brute.step(pos, diam)
    g = orc.step(pos, diam)
    assert np.array_equal(orc.pairs(pos, diam, 0), b["nb"])
    assert np.array_equal(orc.pairs(pos, diam, 1), b["ct"])
    assert np.all(np.abs(g["dp"] - b["dp"]) <= np.maximum(1e-9 * np.abs(b["dp"]), 1e-12))
    # SURVEY.md §8(d).2 statistics for cfg1 (candidates ~39.6, neighbours 6.6, contacts 4.0)
    assert 37 < g["n_cand"].mean() < 42 and 6 < g["n_nb"].mean() < 7.2 and 3.6 < g["n_ct"].mean() < 4.4


def test_mix64_digest(orc):
    # finalizer(0) = 0; finalizer(golden gamma) is the first published SplitMix64 output for seed 0
    assert orc.mix64(0) == 0
    assert orc.mix64(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF


def test_multistep_run_matches_repeated_steps(orc):
    pos, diam = bdm_inputs.random_instance(3, 500, 60.0)
    p3, dp = orc.run(pos, diam, 3)
    q = pos
    for _ in range(3):
        r = orc.step(q, diam)
        q = r["pos_new"]
    assert np.array_equal(p3, q) and np.array_equal(dp, r["dp"])
