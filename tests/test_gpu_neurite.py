"""NEXT-4: neurite elements on the GPU -- sphere-cylinder contacts and spring chains
("the current GPU kernel does not support cylinder geometry yet").
Spheres and distal points must equal the oracle bit for bit after several Jacobi steps."""
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


def trees(rng, n_trees, side):
    """binary trees of 1-7 elements growing from anchors inside the cube, some stretched"""
    Q, d, l0, A, mother, dau = [], [], [], [], [], []
    for _ in range(n_trees):
        root = rng.uniform(-0.4 * side, 0.4 * side, 3)
        base = len(Q)
        k = int(rng.integers(1, 8))
        for j in range(k):
            m = -1 if j == 0 else base + (j - 1) // 2
            P = root if m < 0 else Q[m]
            direc = rng.normal(size=3)
            direc /= np.linalg.norm(direc)
            seg = rng.uniform(3.0, 9.0)
            Q.append(P + direc * seg)
            d.append(rng.uniform(1.0, 4.0))
            l0.append(seg * rng.uniform(0.7, 1.3))
            A.append(root)
            mother.append(m)
            dau.append([-1, -1])
            if m >= 0:
                slot = 0 if dau[m][0] < 0 else 1
                dau[m][slot] = base + j
    return (np.array(Q), np.array(d), np.array(l0), np.array(A), np.array(mother), np.array(dau))


@pytest.mark.parametrize("steps", [1, 4])
def test_neurite_parity(bdm, steps):
    rng = np.random.default_rng(12)
    pos, diam = bdm_inputs.random_instance(41, 2500, 200.0, 8.0, 12.0)
    Q, d, l0, A, mother, dau = trees(rng, 120, 200.0)
    prm = dict(dt=0.2)
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(**prm))
    bdm.bdm_set_neurites(h, Q, d, l0, A, mother, dau, 10.0)
    bdm.bdm_mech_step(h, steps)
    p = bdm.bdm_get_positions(h)
    q, dq = bdm.bdm_get_neurites(h)
    po, qo, dpo, dqo = oracle.neurite_step(pos, diam, Q, d, l0, A, mother, dau[:, 0], dau[:, 1], 10.0,
                                           oracle.params(**prm), steps=steps)
    assert np.array_equal(q, qo) and np.array_equal(dq, dqo)
    assert np.array_equal(p, po)
    assert np.array_equal(bdm.bdm_get_displacements(h), dpo)
    assert np.any(dq != 0.0) and np.any(bdm.bdm_get_displacements(h) != 0.0)


def test_sphere_pushed_by_neurite(bdm):
    """A sphere overlapping a long static element is pushed off perpendicular to the axis."""
    Q = np.array([[40.0, 0.0, 0.0]])
    h = bdm.bdm_init(np.array([[20.0, 9.0, 0.0]]), np.array([10.0]), bdm.bdm_params_default(dt=0.001,
                     max_disp=100.0, adherence=0.0))
    bdm.bdm_set_neurites(h, Q, [10.0], [40.0], np.zeros((1, 3)), [-1], [[-1, -1]], 10.0)
    bdm.bdm_mech_step(h, 1)
    dp = bdm.bdm_get_displacements(h)
    f = 10.0 - 4.0 * np.sqrt(2.5)
    assert abs(dp[0, 1] - 0.001 * f) < 1e-15 and dp[0, 0] == 0.0
    _, dq = bdm.bdm_get_neurites(h)
    assert np.array_equal(dq[0], -dp[0])


def test_grazing_and_crowded_contacts(bdm):
    """Pins the sphere-element contact rows and their fp32 prefilter: spheres grazing a segment's side
    or its distal cap at distance r_s + r_e -+ 1e-9 (contact / none), and hub spheres touched by 8
    radiating elements (more than a contact row holds -> the sphere's own exact search)."""
    pos, diam, Q, d, l0, A, mother = [], [], [], [], [], [], []
    rng = np.random.default_rng(5)
    for k in range(40):
        x0 = np.array([60.0 * k, 0.0, 0.0])
        e = len(Q)
        Q.append(x0 + [20.0, 0.0, 0.0])
        d.append(2.0)
        l0.append(20.0)
        A.append(x0)
        mother.append(-1)
        eps = 1e-9 * (1 if k % 2 else -1)
        pos += [x0 + [10.0, 6.0 + eps, 0.0], x0 + [26.0 + eps, 0.0, 0.0], x0 + [-6.0 - eps, 0.0, 0.0]]
        diam += [10.0, 10.0, 10.0]
        hub = x0 + [0.0, 40.0, 0.0]
        pos.append(hub)
        diam.append(10.0)
        for _ in range(8):
            u = rng.normal(size=3)
            u /= np.linalg.norm(u)
            A.append(hub + 3.0 * u)
            Q.append(hub + 15.0 * u)
            d.append(2.0)
            l0.append(12.0)
            mother.append(-1)
        assert e >= 0
    pos, diam, Q, A = map(np.array, (pos, diam, Q, A))
    d, l0, mother = np.array(d), np.array(l0), np.array(mother)
    dau = np.full((len(Q), 2), -1)
    prm = dict(dt=0.01, adherence=0.0, max_disp=100.0)
    h = bdm.bdm_init(pos, diam, bdm.bdm_params_default(**prm))
    bdm.bdm_set_neurites(h, Q, d, l0, A, mother, dau, 10.0)
    bdm.bdm_mech_step(h, 1)
    dp = bdm.bdm_get_displacements(h)
    q, dq = bdm.bdm_get_neurites(h)
    po, qo, dpo, dqo = oracle.neurite_step(pos, diam, Q, d, l0, A, mother, dau[:, 0], dau[:, 1], 10.0,
                                           oracle.params(**prm), steps=1)
    assert np.array_equal(dp, dpo) and np.array_equal(dq, dqo) and np.array_equal(q, qo)
    touched = np.any(dpo != 0.0, axis=1).reshape(40, 4)
    assert touched[1::2, :3].sum() == 0 and touched[0::2, :3].all()  # +1e-9: none, -1e-9: contact
    assert touched[:, 3].all()
