"""GPU tests of the operator API contract around the hot path (reference oracle.py:50-94).

face_states, reshape-tolerant / dtype-preserving rhs, fused cast + permutation in
pack/unpack, copy-free LSRK4 stepping for any step count, bitwise-reproducible
mass norm (the reference's reruns are byte-identical, pkg/tests/test_cli.py:106-112).
"""

import numpy as np
import pytest
from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import build_oracle_operator, rk4_step  # noqa: E402
from paper_0901_1024_b200 import (CavityMode, Mesh, build_b200_operator, build_reference_element,  # noqa: E402
                                  generate_box_mesh, map_nodes)

TOL = {torch.float32: 1e-5, torch.float64: 1e-12}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _shuffled(seed, cells):
    rng = np.random.default_rng(seed)
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    v = mesh.vertices.copy()
    inner = np.all((v > 1e-9) & (v < 1 - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.05, 0.05, size=(inner.sum(), 3))
    return Mesh(v, np.array([rng.permutation(r) for r in mesh.elements]))


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n", [2, 4, 7])
def test_face_states_match_oracle(dtype, n):
    """u_minus / u_plus in the natural numbering, through element reorder and face-slot permutation."""
    mesh = _shuffled(n, (3, 2, 2))
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(n).normal(size=(6, mesh.num_elements, elem.num_nodes))
    um, up, nrm = op.face_states(state)
    wm, wp, wn = ora.face_states(state)
    assert um.shape == wm.shape == (6, mesh.num_elements, 4, elem.num_face_nodes)
    tol = 0 if dtype == torch.float64 else 3e-7
    assert np.abs(um - wm).max() <= tol * np.abs(wm).max()
    assert rel_l2(up, wp) <= max(tol, 1e-15)
    assert np.allclose(nrm, wn)
    # torch in -> torch out on the device
    tm, tp, _ = op.face_states(torch.as_tensor(state, device="cuda"))
    assert tm.is_cuda and tm.dtype == dtype


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_rhs_reshapes_and_keeps_kind(dtype):
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (2, 2, 2))
    elem = build_reference_element(3)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(3).normal(size=(6, mesh.num_elements, elem.num_nodes))
    want = ora.rhs(state)
    flat = op.rhs(state.reshape(6, -1))          # the reference reshapes (oracle.py:65)
    assert flat.shape == want.shape and flat.dtype == np.float64
    assert rel_l2(flat, want) < TOL[dtype]
    f32 = op.rhs(state.astype(np.float32))       # float32 in -> float32 out (np.empty_like(u))
    assert f32.dtype == np.float32 and rel_l2(f32, want) < 1e-5
    dev = op.rhs(torch.as_tensor(state.ravel(), device="cuda"))
    assert dev.is_cuda and tuple(dev.shape) == want.shape and rel_l2(dev.cpu().numpy(), want) < TOL[dtype]
    with pytest.raises(ValueError):
        op.rhs(state[:, :-1])


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_pack_unpack_cast_and_permutation(dtype):
    """dgm_pack / dgm_unpack: natural float32 or float64, internal element order, padding zero."""
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (3, 3, 2))
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, dtype=dtype, reorder=True)
    assert op._order is not None
    state = np.random.default_rng(0).normal(size=(6, mesh.num_elements, elem.num_nodes))
    for nat in (state, state.astype(np.float32)):
        u = op.to_padded(nat)
        assert op.check_padding(u)
        back64 = op.from_padded(u).cpu().numpy()
        back32 = op.from_padded(u, torch.float32).cpu().numpy()
        assert back32.dtype == np.float32
        ref = nat.astype(np.float32) if dtype == torch.float32 else nat
        assert np.array_equal(back64, ref.astype(np.float64))
        assert np.array_equal(back32, ref.astype(np.float32))
    # the padded layout really is permuted: slot s holds natural element order[s]
    u = op.to_padded(state)
    order = op._order.cpu().numpy()
    got = u[0, : mesh.num_elements, : elem.num_nodes].cpu().numpy()
    want = state[0][order].astype(np.float32 if dtype == torch.float32 else np.float64)
    assert np.array_equal(got, want)
    out = torch.empty((6, mesh.num_elements, elem.num_nodes), dtype=torch.float64, device="cuda")
    assert op.from_padded(u, out=out) is out


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("nsteps,graph", [(1, False), (3, False), (3, True), (11, True)])
def test_advance_any_step_count_without_copies(dtype, nsteps, graph):
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (2, 2, 3))
    elem = build_reference_element(3)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ora = build_oracle_operator(mesh, elem)
    u0 = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0)
    u0 = u0 + 0.05 * np.random.default_rng(1).normal(size=u0.shape)
    dt = 2e-3
    want = u0
    for _ in range(nsteps):
        want = rk4_step(want, 0.0, dt, lambda t, y: ora.rhs(y))
    u = op.to_padded(u0)
    ptr = u.data_ptr()
    op.advance(u, dt, nsteps, use_graph=graph)
    assert u.data_ptr() == ptr
    assert rel_l2(op.from_padded(u).cpu().numpy(), want) < TOL[dtype]
    assert op.check_padding(u)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_mass_norm_is_bitwise_reproducible(dtype):
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (8, 8, 8))   # 3,072 tets: many CTAs
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(5).normal(size=(6, mesh.num_elements, elem.num_nodes))
    u = op.to_padded(state)
    vals = [op.field_energy(u) for _ in range(5)]
    assert len(set(vals)) == 1, vals
    tol = 1e-12 if dtype == torch.float64 else 1e-6   # M u accumulates in the state's precision
    assert abs(vals[0] - ora.energy(op.from_padded(u).cpu().numpy())) <= tol * abs(vals[0])
    # accumulate semantics: *out += value
    acc = torch.full((1,), 1.5, dtype=torch.float64, device="cuda")
    op.mass_norm(u, 1.0, 1.0, out=acc)
    assert abs(float(acc.item()) - 1.5 - 2 * vals[0]) <= 1e-12 * vals[0]


@pytest.mark.gpu
@pytest.mark.parametrize("serial", [False, True])
def test_host_stepper_matches_device_stepping(serial):
    """HostStepper (host-resident state, pipelined per-piece copies) == to_padded / advance / from_padded."""
    import torch

    from paper_0901_1024_b200 import HostStepper

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (4, 3, 3))
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, dtype=torch.float32, device="cuda:0")
    u0 = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0)
    dt = 1e-3
    u = op.to_padded(u0)
    op.advance(u, dt, 3, use_graph=False)
    want = op.from_padded(u).cpu().numpy()
    host = torch.from_numpy(np.ascontiguousarray(u0)).pin_memory()
    energy = torch.zeros(1, dtype=torch.float64).pin_memory()
    st = HostStepper(op, chunks=3, serial=serial)
    for _ in range(3):  # one call per step: the chain continues across calls
        st.step(host, dt, 1, energy_out=energy)
    st.join()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(host.numpy(), want)
    assert energy.item() > 0
    with pytest.raises(ValueError):
        st.step(host[:, :1], dt)


@pytest.mark.gpu
def test_rhs_numpy_pageable_fallback_matches_pinned(monkeypatch):
    """rhs(numpy) through pinned staging and through the pageable fallback give the same array."""
    import torch

    from paper_0901_1024_b200.operator import B200MaxwellOperator

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (3, 3, 2))
    elem = build_reference_element(3)
    u0 = np.random.default_rng(3).normal(size=(6, mesh.num_elements, elem.num_nodes))
    op = build_b200_operator(mesh, elem, dtype=torch.float64, device="cuda:0")
    pinned = op.rhs(u0)
    again = op.rhs(u0)  # cached buffers reused
    monkeypatch.setattr(B200MaxwellOperator, "PINNED_RHS_MAX_BYTES", 0)
    op2 = build_b200_operator(mesh, elem, dtype=torch.float64, device="cuda:0")
    pageable = op2.rhs(u0)
    assert pinned.dtype == np.float64 and pinned.shape == u0.shape
    np.testing.assert_array_equal(pinned, again)
    np.testing.assert_array_equal(pinned, pageable)
    assert op2._pinned_rhs[(u0.dtype.str, torch.float64)] is False
