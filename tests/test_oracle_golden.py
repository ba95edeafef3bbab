"""Pin the CPU oracle to outputs of the real reference (tests/golden, oracle/make_golden.py)."""

import numpy as np
import pytest
from conftest import golden_element, load_golden, rel_l2, rel_max

from oracle import OracleOperator, rk4_step, upwind_bracket
from paper_0901_1024_b200.mesh import Mesh, generate_box_mesh


@pytest.fixture(scope="module")
def c1():
    return load_golden("mesh_c1.npz")


def test_oracle_connectivity_and_vmaps_c1(c1, golden_refelem):
    e3 = golden_element(golden_refelem, 3)
    op = OracleOperator(c1["vertices"], c1["elements"], e3)
    assert np.array_equal(op.interior, c1["interior"])
    assert np.array_equal(op.boundary, c1["boundary"][:, :2])
    assert np.array_equal(op.vmap_minus, c1["vmap_minus"])
    assert np.array_equal(op.vmap_plus, c1["vmap_plus"])
    assert np.array_equal(op.is_boundary, c1["is_boundary"])
    assert np.allclose(op.geo["drdx"], c1["inv_jacobians"], rtol=0, atol=1e-13)
    assert np.allclose(op.geo["normals"], c1["normals"], rtol=0, atol=1e-14)
    assert np.allclose(op.geo["sj"], c1["face_jacobians"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("n", range(1, 7))
def test_oracle_rhs_and_flux_small(golden_refelem, n):
    g = load_golden("rhs_small.npz")
    mesh = generate_box_mesh((1.0, 0.9, 1.1), (1, 2, 1))
    op = OracleOperator(mesh.vertices, mesh.elements, golden_element(golden_refelem, n))
    assert rel_max(op.rhs(g[f"n{n}_state"]), g[f"n{n}_rhs"]) < 1e-13
    # gather_stage scales by area/2 = face_jacobian * FACE_AREAS / 2 (oracle.py:168-189)
    from oracle.dg_oracle import FACE_AREAS

    nfp = golden_element(golden_refelem, n).num_face_nodes
    fac = np.repeat(FACE_AREAS / 2.0, nfp)
    assert rel_max(op.scaled_flux(g[f"n{n}_state"]) * fac, g[f"n{n}_gather"]) < 1e-13


@pytest.mark.parametrize("n", [7, 9])
def test_oracle_rhs_single_tet_high_order(golden_refelem, n):
    g = load_golden("rhs_small.npz")
    mesh = Mesh(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]), np.array([[0, 1, 2, 3]]))
    op = OracleOperator(mesh.vertices, mesh.elements, golden_element(golden_refelem, n))
    assert rel_max(op.rhs(g[f"tet{n}_state"]), g[f"tet{n}_rhs"]) < 1e-12


def test_oracle_c1_random_rhs(c1, golden_refelem):
    g = load_golden("c1_n3.npz")
    op = OracleOperator(c1["vertices"], c1["elements"], golden_element(golden_refelem, 3))
    rnd = np.random.default_rng(0).normal(size=(6, len(c1["elements"]), 20))
    assert rel_max(op.rhs(rnd), g["rhs_random"]) < 1e-13


def test_oracle_c1_ten_steps(c1, golden_refelem):
    """Headline parity config C1: N=3, 1,512 tets, 10 LSRK4 steps (BASELINE.json configs[0])."""
    from paper_0901_1024_b200.maxwell import CavityMode

    g = load_golden("c1_n3.npz")
    e3 = golden_element(golden_refelem, 3)
    op = OracleOperator(c1["vertices"], c1["elements"], e3)
    mesh = Mesh(c1["vertices"], c1["elements"])
    from paper_0901_1024_b200.mesh import map_nodes

    u = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, e3), 0.0)
    energies = [op.energy(u)]
    for _ in range(10):
        u = rk4_step(u, 0.0, float(g["dt"]), lambda t, y: op.rhs(y))
        energies.append(op.energy(u))
    assert rel_l2(u, g["u10"]) < 1e-13
    assert np.allclose(energies, g["energies"], rtol=1e-13, atol=0)


def test_upwind_known_answer():
    g = load_golden("flux_known.npz")
    got = upwind_bracket(g["um"], g["up"], g["normal"])
    assert np.allclose(got, g["bracket"], atol=1e-15)
    assert np.allclose(got, [0.0, -0.5, 0.0, 0.0, 0.0, 0.5])  # test_maxwell.py:86-92


def test_oracle_rk4_rejects_bad_dt():
    with pytest.raises(ValueError):
        rk4_step(np.zeros(2), 0.0, 0.0, lambda t, u: u)
