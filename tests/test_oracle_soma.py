"""Pins for the NEXT-3 oracle (soma clustering: secretion, diffusion, chemotaxis),
against closed forms and invariants of SPEC.md:260-329 (diffusion-field examples and properties)."""
import math

import numpy as np
import pytest


def fp(orc, dims=(20, 20, 20), h=2.0, diff=0.4, decay=0.0, dt=1.0, secretion=1.0, speed=0.5, origin=(0.0, 0.0, 0.0)):
    return orc.fields(h, origin, dims, diff, decay, dt, secretion, speed)


def test_uniform_field_unchanged(orc):
    """uniform field, closed boundary, mu = 0 -> unchanged (zero Laplacian)."""
    f = fp(orc)
    c = np.full((20, 20, 20), 3.25)
    assert np.array_equal(orc.diffuse(f, c), c)


def test_pure_decay_closed_form(orc):
    """SPEC.md:288 / :311: D = 0 -> every node multiplied by (1 - mu dt) each step."""
    f = fp(orc, diff=0.0, decay=0.1)
    rng = np.random.default_rng(0)
    c0 = rng.uniform(0, 5, (20, 20, 20))
    c = c0
    for _ in range(25):
        c = orc.diffuse(f, c)
    assert np.allclose(c, c0 * 0.9 ** 25, rtol=1e-12, atol=0)


def test_mass_conservation_and_maximum_principle(orc):
    """closed boundary, mu = 0: total mass conserved (1e-9 relative over 1000
    steps); max never increases, min never decreases."""
    f = fp(orc, dims=(12, 12, 12), diff=0.6, h=2.0)  # D dt / h^2 = 0.15 <= 1/6
    rng = np.random.default_rng(1)
    c = rng.uniform(0, 1, (12, 12, 12))
    m0, hi, lo = c.sum(), c.max(), c.min()
    for _ in range(1000):
        c2 = orc.diffuse(f, c)
        assert c2.max() <= c.max() + 1e-15 and c2.min() >= c.min() - 1e-15
        c = c2
    assert abs(c.sum() - m0) <= 1e-9 * m0
    assert c.max() <= hi and c.min() >= lo


def test_point_source_heat_kernel(orc):
    """unit mass at the centre of a 41^3 lattice, D dt / h^2 = 0.1, after n steps the
    interior profile matches the free-space heat kernel with variance 2 D n dt (L_inf <= 5% of peak)."""
    n, h, D = 41, 1.0, 0.1
    f = fp(orc, dims=(n, n, n), h=h, diff=D)
    c = np.zeros((n, n, n))
    c[20, 20, 20] = 1.0
    steps = 120
    for _ in range(steps):
        c = orc.diffuse(f, c)
    var = 2 * D * steps
    x = (np.arange(n) - 20.0) * h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    g = np.exp(-(X ** 2 + Y ** 2 + Z ** 2) / (2 * var)) / (2 * math.pi * var) ** 1.5
    inner = (slice(8, 33),) * 3
    assert np.abs(c[inner] - g[inner]).max() <= 0.05 * g.max()


def test_linearity(orc):
    """stepping a sum equals the sum of stepped fields (1e-12)."""
    f = fp(orc, decay=0.05)
    rng = np.random.default_rng(2)
    a, b = rng.uniform(0, 1, (2, 20, 20, 20))
    assert np.allclose(orc.diffuse(f, a + b), orc.diffuse(f, a) + orc.diffuse(f, b), rtol=0, atol=1e-12)


def test_gradient_of_linear_field(orc):
    """linear field c = 3 z -> gradient (0, 0, 3) in the interior; uniform -> 0."""
    f = fp(orc, dims=(10, 10, 10), h=2.0)
    z = np.arange(10) * 2.0
    c = np.broadcast_to(3.0 * z[None, None, :], (10, 10, 10)).copy()
    rng = np.random.default_rng(3)
    for p in rng.uniform(2.5, 15.5, (50, 3)):
        g = orc.gradient_at(f, c, p)
        assert abs(g[0]) < 1e-13 and abs(g[1]) < 1e-13 and abs(g[2] - 3.0) < 1e-13
    assert np.array_equal(orc.gradient_at(f, np.full((10, 10, 10), 2.0), np.array([5.0, 5.0, 5.0])), np.zeros(3))


def test_secretion_nearest_node(orc):
    """secretion adds amount/step to the nearest node; integer counts per node."""
    f = fp(orc, dims=(10, 10, 10), h=2.0, secretion=0.25)
    pos = np.array([[4.0, 4.0, 4.0], [4.9, 3.2, 4.1], [5.1, 4.0, 4.0], [100.0, -50.0, 3.0]])
    types = np.array([0, 0, 0, 1], np.int8)
    c0, c1 = orc.secrete(f, pos, types, np.zeros((10, 10, 10)), np.zeros((10, 10, 10)))
    assert c0[2, 2, 2] == 0.5 and c0[3, 2, 2] == 0.25 and c0.sum() == 0.75
    assert c1[9, 0, 2] == 0.25 and c1.sum() == 0.25  # clamped into the lattice


def test_chemotaxis_moves_speed_along_gradient(orc):
    """S3: an agent in a linear field of its type moves exactly `speed` up the gradient; the other
    type's field does not affect it."""
    f = fp(orc, dims=(10, 10, 10), h=2.0, speed=0.5, diff=0.0, secretion=0.0)
    x = np.arange(10) * 2.0
    c0 = np.broadcast_to((2.0 * x)[:, None, None], (10, 10, 10)).copy()  # grad (2, 0, 0)
    c1 = np.zeros((10, 10, 10))
    pos = np.array([[7.3, 8.1, 9.9], [13.3, 12.1, 5.9]])  # far apart: no contact
    out, _, _, _ = orc.run_soma(pos, np.array([1.0, 1.0]), np.array([0, 1], np.int8), f, 1, c0, c1)
    assert abs(out[0, 0] - (7.3 + 0.5)) < 1e-14 and out[0, 1] == 8.1 and out[0, 2] == 9.9
    assert np.array_equal(out[1], pos[1])  # type 1 sees a flat field


def test_negative_results_clamped(orc):
    """SPEC.md:270 / :286: "negative results clamped to 0".  Closed forms: (a) pure decay with
    mu dt = 1.5 gives c (1 - 1.5) < 0 at every node -> the field is exactly 0 after one step;
    (b) a unit spike with D dt/h^2 = 1/6 and mu dt = 0.5: the spike node would be
    1 + 1 (1/6 (0 - 6) - 0.5) = -0.5 -> 0, its six face neighbours get exactly 1/6 (positive,
    unclamped), everything else stays 0."""
    f = fp(orc, diff=0.0, decay=1.5)
    c = np.random.default_rng(4).uniform(0.1, 5, (20, 20, 20))
    out = orc.diffuse(f, c)
    assert np.array_equal(out, np.zeros_like(c)) and not np.signbit(out).any()
    f = fp(orc, dims=(9, 9, 9), h=3.0, diff=1.5, decay=0.5)  # D dt / h^2 = 1.5 / 9 = 1/6
    c = np.zeros((9, 9, 9))
    c[4, 4, 4] = 1.0
    out = orc.diffuse(f, c)
    assert out[4, 4, 4] == 0.0 and out.min() == 0.0
    expect = 1.0 * (1.5 * (1.0 * (1.0 / 9.0)))  # dt * (D * lap) at a face neighbour, lap = 1/h^2
    for d in [(3, 4, 4), (5, 4, 4), (4, 3, 4), (4, 5, 4), (4, 4, 3), (4, 4, 5)]:
        assert abs(out[d] - 1.0 / 6.0) <= 1e-16 and out[d] == expect
    assert np.count_nonzero(out) == 6


def test_gradient_boundary_cells_one_sided(orc):
    """S3 / SPEC.md:304 "one-sided differences at boundary layers", pinned with closed forms.
    (a) A linear field c = 2x - y + 3z is reproduced exactly by one-sided and central differences
    alike, so the gradient is (2, -1, 3) in the boundary cells and for positions outside the
    lattice (clamped sampling) -- a central-difference factor on a boundary node (0.5/h
    instead of 1/h) would give half the slope there.  (b) c = z^2 (h = 2, 6 nodes): on node 0 the
    one-sided difference is (c1 - c0)/h = h = 2 (central would be undefined, the exact derivative 0);
    on the last node (z = 10) it is (100 - 64)/2 = 18; at the cell midpoint z = 1 the gradient
    interpolates nodes 0 and 1: 0.5 * 2 + 0.5 * (16 - 0)/4 = 3."""
    n, h = 6, 2.0
    f = fp(orc, dims=(n, n, n), h=h)
    x = np.arange(n) * h
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    c = 2.0 * X - Y + 3.0 * Z
    pts = [(0.3, 0.7, 9.9), (9.5, 0.1, 0.0), (0.0, 0.0, 0.0), (10.0, 10.0, 10.0), (1.0, 9.0, 5.0),
           (-3.0, 4.0, 12.5), (15.0, -2.0, 3.3)]
    for p in pts:
        g = orc.gradient_at(f, c, np.array(p))
        assert np.abs(g - np.array([2.0, -1.0, 3.0])).max() <= 1e-13, (p, g)
    c = Z ** 2
    assert orc.gradient_at(f, c, np.array([5.0, 5.0, 0.0]))[2] == 2.0
    assert orc.gradient_at(f, c, np.array([5.0, 5.0, 10.0]))[2] == 18.0
    assert orc.gradient_at(f, c, np.array([5.0, 5.0, 1.0]))[2] == 3.0
    assert orc.gradient_at(f, c, np.array([5.0, 5.0, -4.0]))[2] == 2.0  # clamped below the lattice
