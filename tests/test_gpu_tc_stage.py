"""Tensor-core stage kernel (tcgen05, 3xTF32, A operand in TMEM) against the oracle and the SIMT path."""

import numpy as np
import pytest
from conftest import load_golden, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import build_oracle_operator, rk4_step  # noqa: E402
from paper_0901_1024_b200 import (CavityMode, Mesh, build_b200_operator, build_reference_element,  # noqa: E402
                                  generate_box_mesh, map_nodes)

TC_ORDERS = [1, 2, 3, 4, 5, 6, 7, 8, 9]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _jittered(seed, cells):
    rng = np.random.default_rng(seed)
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    v = mesh.vertices.copy()
    inner = np.all((v > 1e-9) & (v < 1 - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.06, 0.06, size=(inner.sum(), 3))
    return Mesh(v, np.array([rng.permutation(r) for r in mesh.elements]))


@pytest.mark.parametrize("n", TC_ORDERS)
def test_tensor_path_selected_and_rhs_matches_oracle(n):
    mesh = _jittered(30 + n, (4, 3, 3))  # 216 tets: one full tile + a ragged tail tile
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, dtype=torch.float32, path="tensor")
    assert op.path == "tensor"
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(n).normal(size=(6, mesh.num_elements, elem.num_nodes))
    err = rel_l2(op.rhs(state), ora.rhs(state))
    print(f"N={n} tensor rhs rel L2 {err:.2e}")
    assert err < 1e-5


@pytest.mark.parametrize("n", TC_ORDERS)
def test_tensor_and_simt_paths_agree_on_steps(n):
    mesh = _jittered(40 + n, (3, 3, 5))
    elem = build_reference_element(n)
    tc = build_b200_operator(mesh, elem, path="tensor")
    si = build_b200_operator(mesh, elem, path="simt")
    assert si.path == "simt"
    u0 = np.random.default_rng(5).normal(size=(6, mesh.num_elements, elem.num_nodes))
    a, b = tc.to_padded(u0), si.to_padded(u0)
    tc.advance(a, 1e-3, 3, use_graph=False)
    si.advance(b, 1e-3, 3, use_graph=False)
    assert tc.check_padding(a)
    assert rel_l2(tc.from_padded(a).cpu().numpy(), si.from_padded(b).cpu().numpy()) < 1e-5


def test_tensor_path_c1_ten_steps_vs_reference():
    g = load_golden("c1_n3.npz")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (6, 6, 7))
    elem = build_reference_element(3)
    op = build_b200_operator(mesh, elem, path="tensor")
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    op.advance(u, float(g["dt"]), 10)
    err = rel_l2(op.from_padded(u).cpu().numpy(), g["u10"])
    print(f"C1 tensor 10 steps rel L2 {err:.2e}")
    assert err < 1e-5


def test_tensor_path_n4_box_vs_reference():
    g = load_golden("box3_n4.npz")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (3, 3, 3))
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, path="tensor")
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    op.advance(u, float(g["dt"]), 10)
    assert rel_l2(op.from_padded(u).cpu().numpy(), g["u10"]) < 1e-5


def test_tensor_path_element_subranges():
    """Interior/boundary split launches (multi-GPU) on arbitrary, odd element ranges."""
    mesh = _jittered(7, (4, 4, 3))
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, path="tensor")
    ora = build_oracle_operator(mesh, elem)
    u0 = np.random.default_rng(9).normal(size=(6, mesh.num_elements, elem.num_nodes))
    u = op.to_padded(u0)
    out = torch.zeros_like(u)
    k = mesh.num_elements
    for lo, hi in [(0, 37), (37, 200), (200, k)]:
        op.rhs_padded(u, out, lo, hi)
    assert rel_l2(op.from_padded(out).cpu().numpy(), ora.rhs(u0)) < 1e-5
    want = rk4_step(u0, 0.0, 1e-3, lambda t, y: ora.rhs(y))
    op.advance(u, 1e-3, 1, use_graph=False)
    assert rel_l2(op.from_padded(u).cpu().numpy(), want) < 1e-5


@pytest.mark.parametrize("n", [2, 4, 7])
def test_locality_reordered_operator_matches_oracle(n):
    """build_b200_operator(reorder=True): internal Morton numbering, natural-order API unchanged."""
    mesh = _jittered(60 + n, (4, 3, 3))
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, reorder=True)
    plain = build_b200_operator(mesh, elem)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(n).normal(size=(6, mesh.num_elements, elem.num_nodes))
    assert rel_l2(op.rhs(state), ora.rhs(state)) < 1e-5
    a, b = op.to_padded(state), plain.to_padded(state)
    op.advance(a, 1e-3, 3, use_graph=False)
    plain.advance(b, 1e-3, 3, use_graph=False)
    assert rel_l2(op.from_padded(a).cpu().numpy(), plain.from_padded(b).cpu().numpy()) < 1e-5
    assert abs(op.field_energy(a) - plain.field_energy(b)) <= 1e-5 * plain.field_energy(b)


@pytest.mark.parametrize("n", [3, 4, 6, 9])
def test_face_slot_order_is_invisible(n):
    """face_slots=True (bank-spread node order inside each face) vs the natural order: same RHS,
    same natural-order surface flux, same steps; also on the fp64 SIMT path.  The natural plan is
    created second with fewer codes (less smem): it must not shrink the first plan's smem limit."""
    mesh = _jittered(80 + n, (4, 3, 3))
    elem = build_reference_element(n)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(n).normal(size=(6, mesh.num_elements, elem.num_nodes))
    slot = build_b200_operator(mesh, elem, path="tensor", face_slots=True)
    nat = build_b200_operator(mesh, elem, path="tensor", face_slots=False)
    assert slot._slot_inv is not None and nat._slot_inv is None
    assert rel_l2(slot.rhs(state), ora.rhs(state)) < 1e-5
    sa, sb = slot.to_padded(state), nat.to_padded(state)
    assert rel_l2(slot.surface_flux(sa).cpu().numpy(), nat.surface_flux(sb).cpu().numpy()) < 1e-6
    slot.advance(sa, 1e-3, 3, use_graph=False)
    nat.advance(sb, 1e-3, 3, use_graph=False)
    assert rel_l2(slot.from_padded(sa).cpu().numpy(), nat.from_padded(sb).cpu().numpy()) < 1e-5
    f64 = build_b200_operator(mesh, elem, dtype=torch.float64, face_slots=True)
    assert rel_l2(f64.rhs(state), ora.rhs(state)) < 1e-12
