"""GPU parity: the sm_100a kernels (through libdgm.so's C ABI) against the CPU oracle and golden data.

Tolerances (BASELINE.json north_star): fp32 relative L2 <= 1e-5, fp64 <= 1e-12
for fields after a fixed number of steps; integer maps bit-exact (CPU tests).
"""

import numpy as np
import pytest
from conftest import golden_element, load_golden, rel_l2, rel_max

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import OracleOperator, build_oracle_operator, rk4_step  # noqa: E402
from paper_0901_1024_b200 import (CavityMode, Mesh, build_b200_operator, build_reference_element,  # noqa: E402
                                  compute_geometry, generate_box_mesh, map_nodes, stable_dt)
from paper_0901_1024_b200 import rk4_step as device_rk4_step  # noqa: E402
from paper_0901_1024_b200.maxwell import Material  # noqa: E402

TOL = {torch.float32: 1e-5, torch.float64: 1e-12}
RHS_TOL = {torch.float32: 1e-5, torch.float64: 1e-13}
DTYPES = [torch.float32, torch.float64]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _jittered(seed=0, cells=(2, 2, 2)):
    rng = np.random.default_rng(seed)
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    v = mesh.vertices.copy()
    inner = np.all((v > 1e-9) & (v < 1 - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.06, 0.06, size=(inner.sum(), 3))
    return Mesh(v, np.array([rng.permutation(r) for r in mesh.elements]))


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", range(1, 10))
def test_rhs_matches_oracle_all_orders(dtype, n):
    mesh = _jittered(n, (2, 2, 1)) if n <= 6 else _jittered(n, (1, 1, 1))
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(100 + n).normal(size=(6, mesh.num_elements, elem.num_nodes))
    got = op.rhs(state)
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    err = rel_l2(got, ora.rhs(state))
    print(f"N={n} {dtype} rhs rel L2 {err:.3e}")
    assert err < RHS_TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", range(1, 7))
def test_rhs_matches_reference_golden(golden_refelem, dtype, n):
    g = load_golden("rhs_small.npz")
    mesh = generate_box_mesh((1.0, 0.9, 1.1), (1, 2, 1))
    op = build_b200_operator(mesh, build_reference_element(n), dtype=dtype)
    assert rel_max(op.rhs(g[f"n{n}_state"]), g[f"n{n}_rhs"]) < 10 * RHS_TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [1, 3, 4, 6, 8])
def test_stage_kernels_match_oracle_stages(dtype, n):
    mesh = _jittered(7 + n, (2, 1, 2))
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(n).normal(size=(6, mesh.num_elements, elem.num_nodes))
    u = op.to_padded(state)
    assert rel_l2(op.from_padded(op.volume_padded(u)).cpu().numpy(), ora.volume(state)) < RHS_TOL[dtype]
    assert rel_l2(op.surface_flux(u).cpu().numpy(), ora.scaled_flux(state)) < RHS_TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_c1_ten_steps_vs_reference(dtype):
    """C1 (BASELINE configs[0]): N=3, cavity (1,1,1), 1,512 tets, 10 LSRK4 steps."""
    g = load_golden("c1_n3.npz")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (6, 6, 7))
    elem = build_reference_element(3)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    dt = stable_dt(mesh, compute_geometry(mesh), 3)
    assert dt == float(g["dt"])
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    energies = [op.field_energy(u)]
    for _ in range(10):
        op.step(u, dt)
        energies.append(op.field_energy(u))
    got = op.from_padded(u).cpu().numpy()
    assert rel_l2(got, g["u10"]) < TOL[dtype]
    assert np.allclose(energies, g["energies"], rtol=TOL[dtype], atol=0)
    assert op.check_padding(u)
    assert rel_max(op.rhs(np.random.default_rng(0).normal(size=got.shape)), g["rhs_random"]) < 10 * RHS_TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_n4_box_ten_steps_graph_vs_reference(dtype):
    g = load_golden("box3_n4.npz")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (3, 3, 3))
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    u0 = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0)
    a = op.to_padded(u0)
    op.advance(a, float(g["dt"]), 10, use_graph=True)
    b = op.to_padded(u0)
    op.advance(b, float(g["dt"]), 10, use_graph=False)
    assert torch.equal(a, b)  # graph replay is bit-identical to eager launches
    assert rel_l2(op.from_padded(a).cpu().numpy(), g["u10"]) < TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_odd_step_counts_and_generic_rk4(dtype):
    mesh = _jittered(5)
    elem = build_reference_element(2)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ora = build_oracle_operator(mesh, elem)
    u0 = np.random.default_rng(3).normal(size=(6, mesh.num_elements, elem.num_nodes))
    want = u0
    for _ in range(5):
        want = rk4_step(want, 0.0, 2e-3, lambda t, y: ora.rhs(y))
    u = op.to_padded(u0)
    op.advance(u, 2e-3, 5)  # 2 graph pairs + 1 eager step
    assert rel_l2(op.from_padded(u).cpu().numpy(), want) < TOL[dtype]
    # reference-signature stepper on device tensors (rhs_fn = fused RHS kernel)
    v = op.to_padded(u0)
    for _ in range(5):
        v = device_rk4_step(v, 0.0, 2e-3, lambda t, y: op.rhs_padded(y))
    assert rel_l2(op.from_padded(v).cpu().numpy(), want) < TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [3, 7, 9])
def test_material_constants(dtype, n):
    """eps, mu != 1 on every lane mapping of the tensor kernel (N=3: E|H tiles, 7: comp-major, 9: one tile)."""
    mesh = _jittered(2) if n <= 3 else _jittered(2, (2, 1, 1))
    elem = build_reference_element(n)
    mat = Material(permittivity=2.0, permeability=0.5)
    op = build_b200_operator(mesh, elem, mat, dtype=dtype)
    ora = OracleOperator(mesh.vertices, mesh.elements, elem, eps=2.0, mu=0.5)
    state = np.random.default_rng(9).normal(size=(6, mesh.num_elements, elem.num_nodes))
    assert rel_l2(op.rhs(state), ora.rhs(state)) < RHS_TOL[dtype]


def test_constant_h_is_steady():
    mesh = generate_box_mesh((1, 1, 1), (2, 2, 2))
    elem = build_reference_element(3)
    op = build_b200_operator(mesh, elem, dtype=torch.float64)
    nat = np.zeros((6, mesh.num_elements, elem.num_nodes))
    nat[3:] = 0.7
    assert np.abs(op.rhs(nat)).max() < 1e-12


def test_torch_in_torch_out_and_errors():
    mesh = generate_box_mesh((1, 1, 1), (1, 1, 1))
    elem = build_reference_element(2)
    op = build_b200_operator(mesh, elem)
    st = torch.randn(6, 6, elem.num_nodes, dtype=torch.float64)
    out = op.rhs(st)
    assert isinstance(out, torch.Tensor) and out.device == st.device
    with pytest.raises(ValueError):
        op.rhs(np.zeros((6, 5, elem.num_nodes)))
    with pytest.raises(ValueError):
        op.advance(op.empty_state(), 0.0)
    with pytest.raises(ValueError):
        op.rhs_padded(torch.zeros(6, 6, op.np_stride, device="cuda", dtype=torch.float64))  # f32 expected
    with pytest.raises(ValueError):
        build_b200_operator(mesh, elem, dtype=torch.float16)


def test_large_mesh_properties_fp32():
    """Size-independent properties at ~100k tets: linearity, energy decay, padding invariant."""
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (26, 26, 26))
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, dtype=torch.float32)
    gen = torch.Generator(device="cuda").manual_seed(0)
    shape = (6, mesh.num_elements, elem.num_nodes)
    x = torch.randn(shape, generator=gen, device="cuda", dtype=torch.float64)
    y = torch.randn(shape, generator=gen, device="cuda", dtype=torch.float64)
    rx = op.rhs_padded(op.to_padded(x))
    ry = op.rhs_padded(op.to_padded(y))
    rxy = op.rhs_padded(op.to_padded(2.0 * x - 3.0 * y))
    lin = (rxy - (2.0 * rx - 3.0 * ry)).norm() / rxy.norm()
    assert lin.item() < 1e-5
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    dt = stable_dt(mesh, compute_geometry(mesh), 4)
    e_prev = op.field_energy(u)
    for _ in range(4):
        op.advance(u, dt, 5)
        e = op.field_energy(u)
        assert e <= e_prev * (1 + 1e-6)
        e_prev = e
    assert op.check_padding(u)


def test_workspaces_on_two_streams_match_default_path():
    """op.advance(..., workspace=) on separate CUDA streams (the bench's e2e pattern) == the default path."""
    mesh = _jittered(3, (3, 2, 2))
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, dtype=torch.float32)
    u0 = np.random.default_rng(11).normal(size=(6, mesh.num_elements, elem.num_nodes))
    ref = op.to_padded(u0)
    op.advance(ref, 1e-3, 3, use_graph=False)
    streams = [torch.cuda.Stream() for _ in range(2)]
    works = [op.workspace() for _ in range(2)]
    outs = [op.empty_state() for _ in range(2)]
    for j in range(2):
        with torch.cuda.stream(streams[j]):
            op.to_padded(u0, out=outs[j])
            op.advance(outs[j], 1e-3, 3, use_graph=(j == 1), workspace=works[j])
    torch.cuda.synchronize()
    for j in range(2):
        assert torch.equal(outs[j], ref)


def test_stage_stats_count_kernel_launches():
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (2, 2, 2))
    elem = build_reference_element(3)
    op = build_b200_operator(mesh, elem)
    u = op.to_padded(np.random.default_rng(2).normal(size=(6, mesh.num_elements, elem.num_nodes)))
    op.collect_stats = True
    op.advance(u, 1e-3, 2, use_graph=False)
    op.rhs_padded(u)
    st = op.stage_stats
    assert st["lsrk_stage"].launches == 10 and st["rhs"].launches == 1
    assert op.total_stats().launches == 11 and op.total_stats().ms > 0
    op.reset_stats()
    assert op.stage_stats == {}
