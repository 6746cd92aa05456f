"""Pins for the NEXT-2 oracle (cell growth and division): closed forms and the
2^n doubling oracle of SPEC.md:101, volume conservation of SPEC.md:88-91 / SPEC.md:117."""
import math

import numpy as np
import pytest

import bdm_inputs


def test_growth_below_threshold_is_linear(orc):
    pos, diam = bdm_inputs.random_instance(1, 50, 300.0, 6.0, 8.0)
    p2, d2 = orc.grow_divide(pos, diam, 0.5, 100.0, 1, 0)
    assert len(d2) == 50 and np.array_equal(p2, pos) and np.array_equal(d2, diam + 0.5)


def test_division_conserves_volume_and_touches(orc):
    """SPEC.md:88 example: d=10, ratio 0.5 -> both 10*(0.5)^(1/3) = 7.937 um; total volume conserved
    (1e-12 relative); the two daughters touch (centre distance = daughter diameter)."""
    pos = np.array([[1.0, 2.0, 3.0]])
    p2, d2 = orc.grow_divide(pos, np.array([9.5]), 0.5, 10.0, 7, 3)
    assert len(d2) == 2
    assert abs(d2[0] - 10.0 * 0.5 ** (1.0 / 3.0)) < 1e-14 and d2[0] == d2[1]
    v0 = math.pi / 6 * 10.0 ** 3
    v1 = 2 * math.pi / 6 * d2[0] ** 3
    assert abs(v1 - v0) <= 1e-12 * v0
    dist = np.linalg.norm(p2[0] - p2[1])
    assert abs(dist - d2[0]) < 1e-13
    mid = 0.5 * (p2[0] + p2[1])  # symmetric about the parent's centre
    assert np.all(np.abs(mid - pos[0]) < 1e-14)


@pytest.mark.parametrize("steps", [1, 2, 3, 4])
def test_doubling_oracle(orc, steps):
    """one agent dividing every step -> population 2^n; here with mechanics between
    divisions (the daughters touch, so no force acts at division time)."""
    pos = np.array([[0.0, 0.0, 0.0]])
    p, d, _ = orc.run_growth(pos, np.array([10.0]), steps, growth=0.0, div_diam=1.0, seed=2)
    assert len(d) == 2 ** steps
    # every division halves the volume: all diameters equal 10 * 2^(-steps/3) (up to rounding)
    assert np.all(np.abs(d - 10.0 * 2.0 ** (-steps / 3.0)) < 1e-12)


def test_daughter_ids_follow_id_order(orc):
    pos = np.array([[0.0, 0, 0], [100.0, 0, 0], [200.0, 0, 0], [300.0, 0, 0]])
    diam = np.array([11.9, 8.0, 12.5, 12.1])  # ids 0, 2, 3 divide (>= 12 after +0.2)
    p2, d2 = orc.grow_divide(pos, diam, 0.2, 12.0, 5, 0)
    assert len(d2) == 7
    # daughters 4, 5, 6 belong to mothers 0, 2, 3 (ascending id): each sits next to its mother
    for dau, mom in ((4, 0), (5, 2), (6, 3)):
        assert abs(np.linalg.norm(p2[dau] - p2[mom]) - d2[mom]) < 1e-12
    assert d2[1] == 8.2


def test_direction_is_deterministic_and_isotropic(orc):
    n = 4000
    pos = np.zeros((n, 3)) + np.arange(n)[:, None] * np.array([50.0, 0.0, 0.0])
    p2, d2 = orc.grow_divide(pos, np.full(n, 12.0), 0.0, 12.0, 11, 9)
    u = (p2[n:] - p2[:n]) / d2[:n, None]
    assert np.allclose(np.linalg.norm(u, axis=1), 1.0, atol=1e-14)
    assert np.all(np.abs(u.mean(axis=0)) < 0.05)  # isotropic: mean direction ~ 0
    p3, _ = orc.grow_divide(pos, np.full(n, 12.0), 0.0, 12.0, 11, 9)
    assert np.array_equal(p2, p3)
