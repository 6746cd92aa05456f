"""Pins for the NEXT-4 oracle (sphere-cylinder contacts and neurite spring chains)
from SPEC.md:230-238 and SPEC.md:377-386 worked examples and properties."""
import math

import numpy as np

F = float(np.float64(10.0 - 4.0 * math.sqrt(2.5)))  # f(delta = 1) for r = 2.5 (closed form, golden file)


def chain(n_el, seg=5.0, rest=5.0, d=2.0):
    """straight chain along +x from an anchor at the origin"""
    Q = np.array([[seg * (e + 1), 0.0, 0.0] for e in range(n_el)])
    anchor = np.zeros((n_el, 3))
    mother = np.arange(n_el) - 1
    c1 = np.array([e + 1 if e + 1 < n_el else -1 for e in range(n_el)])
    c2 = -np.ones(n_el, int)
    return Q, np.full(n_el, d), np.full(n_el, rest), anchor, mother, c1, c2


def no_spheres():
    return np.zeros((0, 3)), np.zeros(0)


def test_chain_at_rest(orc):
    """chain at rest (actual = resting everywhere) -> all displacements zero."""
    Q, d, l0, A, m, c1, c2 = chain(4)
    _, Q2, _, dQ = orc.neurite_step(*no_spheres(), Q, d, l0, A, m, c1, c2, 10.0)
    assert np.all(dQ == 0.0) and np.array_equal(Q2, Q)


def test_single_element_stretched_twice(orc):
    """one element stretched to 2x resting -> restoring force k_s * 1.0 pulling the distal
    point toward the proximal one (here dt = 0.01, no clamp, no adherence: dQ = -0.1 x_hat)."""
    Q, d, l0, A, m, c1, c2 = chain(1, seg=10.0, rest=5.0)
    prm = orc.params(dt=0.01, max_disp=100.0, adherence=0.0)
    _, _, _, dQ = orc.neurite_step(*no_spheres(), Q, d, l0, A, m, c1, c2, 10.0, prm)
    assert abs(dQ[0, 0] + 0.1) < 1e-15 and dQ[0, 1] == 0.0 and dQ[0, 2] == 0.0


def test_spring_transmits_to_mother(orc):
    """PAPER.md:410 springs "transmit forces along the chain": a stretched daughter pulls its
    mother's distal point forward with the same tension."""
    Q, d, l0, A, m, c1, c2 = chain(2)
    Q[1, 0] = 15.0  # daughter stretched to 2x
    prm = orc.params(dt=0.01, max_disp=100.0, adherence=0.0)
    _, _, _, dQ = orc.neurite_step(*no_spheres(), Q, d, l0, A, m, c1, c2, 10.0, prm)
    assert abs(dQ[0, 0] - 0.1) < 1e-15 and abs(dQ[1, 0] + 0.1) < 1e-15


def test_sphere_on_bisector(orc):
    """sphere centred on the perpendicular bisector of a long element with overlap delta
    -> force perpendicular to the axis with the sphere law's magnitude; the reaction goes to the
    distal point (Newton's third law, bit-exact).  r_s = 5, r_e = 5 (d = 10): r = 2.5, delta = 1."""
    Q, d, l0, A, m, c1, c2 = chain(1, seg=40.0, rest=40.0, d=10.0)
    pos = np.array([[20.0, 9.0, 0.0]])
    prm = orc.params(dt=0.001, max_disp=100.0, adherence=0.0)
    p2, Q2, dp, dQ = orc.neurite_step(pos, np.array([10.0]), Q, d, l0, A, m, c1, c2, 10.0, prm)
    assert abs(dp[0, 1] - 0.001 * F) < 1e-15 and dp[0, 0] == 0.0 and dp[0, 2] == 0.0
    assert abs(dQ[0, 1] + 0.001 * F) < 1e-15
    assert np.array_equal(dp[0] * -1.0, dQ[0])


def test_force_constant_along_interior(orc):
    """sweeping the sphere along the axis, the force magnitude stays constant while the
    closest point is interior, and vanishes beyond the ends."""
    Q, d, l0, A, m, c1, c2 = chain(1, seg=40.0, rest=40.0, d=10.0)
    prm = orc.params(dt=0.001, max_disp=100.0, adherence=0.0)
    mags = []
    for x in np.linspace(2.0, 38.0, 13):
        _, _, dp, _ = orc.neurite_step(np.array([[x, 9.0, 0.0]]), np.array([10.0]), Q, d, l0, A, m, c1, c2, 10.0, prm)
        mags.append(np.linalg.norm(dp[0]))
    assert np.ptp(mags) < 1e-15 and abs(mags[0] - 0.001 * F) < 1e-15
    _, _, dp, _ = orc.neurite_step(np.array([[60.0, 9.0, 0.0]]), np.array([10.0]), Q, d, l0, A, m, c1, c2, 10.0, prm)
    assert np.all(dp == 0.0)


def test_chain_relaxes(orc):
    """a 3-element chain with the middle stretched relaxes to strains < 1e-3."""
    Q, d, l0, A, m, c1, c2 = chain(3)
    Q[1:, 0] += 3.0  # middle element 8 long for rest 5
    prm = orc.params(dt=0.05, max_disp=1.0, adherence=0.0)
    _, Qn, _, _ = orc.neurite_step(*no_spheres(), Q, d, l0, A, m, c1, c2, 10.0, prm, steps=400)
    P = np.vstack([np.zeros(3), Qn[:-1]])
    strain = np.abs(np.linalg.norm(Qn - P, axis=1) - 5.0) / 5.0
    assert strain.max() < 1e-3
