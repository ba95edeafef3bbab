"""The v2 tensor-core stage kernel (dgm_tc2.cuh, path "tensor2", N <= 4 fp32) against the oracle.

Same bar as the v1 kernel (tests/test_gpu_parity.py, test_gpu_tc_stage.py): fp32 relative L2
<= 1e-5 on RHS and after LSRK4 steps; partial tiles, element sub-ranges, materials, padding.
"""

import numpy as np
import pytest
from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import build_oracle_operator, rk4_step  # noqa: E402
from paper_0901_1024_b200 import (CavityMode, Mesh, build_b200_operator, build_reference_element,  # noqa: E402
                                  compute_geometry, generate_box_mesh, map_nodes, stable_dt)
from paper_0901_1024_b200.maxwell import Material  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _jittered(seed, cells):
    rng = np.random.default_rng(seed)
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    v = mesh.vertices.copy()
    inner = np.all((v > 1e-9) & (v < 1 - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.04, 0.04, size=(inner.sum(), 3))
    return Mesh(v, np.array([rng.permutation(r) for r in mesh.elements]))


@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("cells", [(1, 1, 1), (3, 2, 2), (6, 5, 4)])
def test_tc2_rhs_matches_oracle(n, cells):
    mesh = _jittered(n + 10 * cells[0], cells)
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, path="tensor2")
    assert op.path == "tensor2"
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(n).normal(size=(6, mesh.num_elements, elem.num_nodes))
    err = rel_l2(op.rhs(state), ora.rhs(state))
    print(f"tc2 N={n} K={mesh.num_elements} rhs rel L2 {err:.2e}")
    assert err < 1e-5


@pytest.mark.parametrize("n", [3, 4])
def test_tc2_steps_and_padding(n):
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (5, 4, 4))   # 480 tets: 7 full tiles + a partial one
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, path="tensor2")
    ora = build_oracle_operator(mesh, elem)
    u0 = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0)
    u0 = u0 + 0.05 * np.random.default_rng(3).normal(size=u0.shape)
    dt = stable_dt(mesh, compute_geometry(mesh), n)
    want = u0
    for _ in range(10):
        want = rk4_step(want, 0.0, dt, lambda t, y: ora.rhs(y))
    u = op.to_padded(u0)
    op.advance(u, dt, 10)
    assert op.check_padding(u)
    err = rel_l2(op.from_padded(u).cpu().numpy(), want)
    print(f"tc2 N={n} 10 steps rel L2 {err:.2e}")
    assert err < 1e-5


def test_tc2_matches_v1_and_subranges():
    mesh = _jittered(5, (6, 6, 5))
    elem = build_reference_element(4)
    op2 = build_b200_operator(mesh, elem, path="tensor2", reorder=False)
    op1 = build_b200_operator(mesh, elem, path="tensor", reorder=False)
    state = torch.randn((6, mesh.num_elements, elem.num_nodes), device="cuda", dtype=torch.float64)
    u2, u1 = op2.to_padded(state), op1.to_padded(state)
    r2, r1 = op2.rhs_padded(u2), op1.rhs_padded(u1)
    # the face-slot orders differ, the natural results must not
    assert rel_l2(op2.from_padded(r2).cpu().numpy(), op1.from_padded(r1).cpu().numpy()) < 2e-6
    # element sub-ranges (the multi-GPU interior / boundary launches): rows outside stay untouched
    k = mesh.num_elements
    out = torch.full_like(r2, 7.0)
    for lo, hi in ((0, 37), (37, 100), (100, k)):
        op2.rhs_padded(u2, out, lo, hi)
    assert torch.equal(out, r2)


def test_tc2_material():
    mesh = _jittered(9, (3, 3, 2))
    elem = build_reference_element(4)
    mat = Material(permittivity=2.5, permeability=0.7)
    op = build_b200_operator(mesh, elem, mat, path="tensor2")
    ora = build_oracle_operator(mesh, elem, 2.5, 0.7)
    state = np.random.default_rng(1).normal(size=(6, mesh.num_elements, elem.num_nodes))
    assert rel_l2(op.rhs(state), ora.rhs(state)) < 1e-5
