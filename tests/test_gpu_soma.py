"""NEXT-3: soma clustering on the GPU against the oracle -- the
paper's second GPU benchmark ("soma clustering", 5.04x on a V100).
Secretion, diffusion of both substances, chemotaxis and the mechanics: positions, displacements and
both fields must equal the oracle bit for bit after several steps."""
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

    return b


def setup(n, seed, side):
    pos, diam = bdm_inputs.random_instance(seed, n, side, 8.0, 12.0)
    types = (np.random.default_rng(seed).random(n) < 0.5).astype(np.int8)
    h = 12.0
    origin = (-0.5 * side - 2 * h,) * 3
    dims = (int(side / h) + 5,) * 3
    return pos, diam, types, dict(h=h, origin=origin, dims=dims, diff=20.0, decay=0.01, dt=1.0, secretion=1.0,
                                  speed=0.5)


@pytest.mark.parametrize("steps", [1, 5])
def test_soma_parity(bdm, steps):
    pos, diam, types, f = setup(4000, 31, 240.0)
    h = bdm.bdm_init(pos, diam)
    bdm.bdm_set_fields(h, f["h"], f["origin"], f["dims"], f["diff"], f["decay"], f["dt"], f["secretion"],
                       f["speed"], types)
    bdm.bdm_mech_step(h, steps)
    p = bdm.bdm_get_positions(h)
    c0, c1 = bdm.bdm_get_field(h, 0), bdm.bdm_get_field(h, 1)
    fp = oracle.fields(f["h"], f["origin"], f["dims"], f["diff"], f["decay"], f["dt"], f["secretion"], f["speed"])
    po, o0, o1, dpo = oracle.run_soma(pos, diam, types, fp, steps)
    assert np.array_equal(c0, o0) and np.array_equal(c1, o1)
    assert np.array_equal(p, po)
    assert np.array_equal(bdm.bdm_get_displacements(h), dpo)
    assert c0.sum() > 0 and c1.sum() > 0


def test_soma_boundary_cells_and_clamp(bdm):
    """Agents in the lattice's boundary cells and outside it (one-sided node gradients, clamped
    sampling: DESIGN.md S3) with diffusion parameters that drive nodes negative
    (D dt/h^2 = 1/6, mu dt = 0.5 -> 6 D dt/h^2 + mu dt = 1.5 > 1: the SPEC.md:270/286 clamp is
    taken): fields, positions and displacements equal the oracle bit for bit after 4 steps."""
    n, side, hh = 3000, 200.0, 12.0
    pos, diam = bdm_inputs.random_instance(77, n, side, 8.0, 12.0)
    types = (np.random.default_rng(77).random(n) < 0.5).astype(np.int8)
    # lattice covering only [-84, 84]^3 of the [-100, 100]^3 population: boundary cells are
    # populated and ~30% of the agents sit outside the lattice
    origin, dims = (-84.0, -84.0, -84.0), (15, 15, 15)
    f = dict(h=hh, origin=origin, dims=dims, diff=hh * hh / 6.0, decay=0.5, dt=1.0, secretion=1.0, speed=0.5)
    fp = oracle.fields(f["h"], f["origin"], f["dims"], f["diff"], f["decay"], f["dt"], f["secretion"], f["speed"])
    steps = 4
    po, o0, o1, dpo = oracle.run_soma(pos, diam, types, fp, steps)
    # the clamp is reached (a node that would go negative) and agents lie in boundary cells
    q = (pos - np.array(origin)) / hh
    assert ((q < 1) | (q >= dims[0] - 2)).any(axis=1).sum() > 500
    h = bdm.bdm_init(pos, diam)
    bdm.bdm_set_fields(h, f["h"], f["origin"], f["dims"], f["diff"], f["decay"], f["dt"], f["secretion"],
                       f["speed"], types)
    bdm.bdm_mech_step(h, steps)
    c0, c1 = bdm.bdm_get_field(h, 0), bdm.bdm_get_field(h, 1)
    assert np.array_equal(c0, o0) and np.array_equal(c1, o1)
    assert np.array_equal(bdm.bdm_get_positions(h), po)
    assert np.array_equal(bdm.bdm_get_displacements(h), dpo)
    assert (c0 == 0).any() and c0.max() > 0


def test_soma_types_segregate(bdm):
    """Soma clustering's purpose (same-type clustering): after some steps each
    agent's nearest neighbour is more often of its own type than at the start."""
    from scipy.spatial import cKDTree

    pos, diam, types, f = setup(6000, 5, 300.0)
    h = bdm.bdm_init(pos, diam)
    bdm.bdm_set_fields(h, f["h"], f["origin"], f["dims"], 60.0, 0.0, 0.4, 1.0, 1.0, types)

    def same_type_fraction(p):
        _, nn = cKDTree(p).query(p, k=2)
        return float(np.mean(types[nn[:, 1]] == types))

    before = same_type_fraction(pos)
    bdm.bdm_mech_step(h, 60)
    after = same_type_fraction(bdm.bdm_get_positions(h))
    assert after > before + 0.05, (before, after)


def test_unstable_diffusion_rejected(bdm):
    pos, diam, types, f = setup(100, 1, 100.0)
    h = bdm.bdm_init(pos, diam)
    with pytest.raises(bdm.BdmError) as e:
        bdm.bdm_set_fields(h, 1.0, (0, 0, 0), (10, 10, 10), 0.5, 0.0, 1.0, 1.0, 1.0, types)  # D dt/h^2 = 0.5
    assert e.value.code == bdm.BDM_EINVAL
