"""The reference's known-answer tests of this path, restated on the B200 operator (C-ABI kernels).

* constant field => zero volume term          (test_kernels.py:140-147)
* linear field => exact curls                  (test_kernels.py:149-155, unit gradient)
* continuous linear field => zero interior flux (test_kernels.py:264-282)
* two-sided flux conservation                  (test_maxwell.py:94-104), over every glued node pair
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_0901_1024_b200 import (Mesh, build_b200_operator, build_reference_element,  # noqa: E402
                                  generate_box_mesh, map_nodes)
from paper_0901_1024_b200.maxwell import flux  # noqa: E402

TOL = {torch.float32: 2e-5, torch.float64: 1e-11}
DTYPES = [torch.float32, torch.float64]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _mesh(seed, cells=(2, 2, 2)):
    rng = np.random.default_rng(seed)
    mesh = generate_box_mesh((1.0, 0.8, 1.3), cells)
    v = mesh.vertices.copy()
    inner = np.all((v > 1e-9) & (v < np.array([1.0, 0.8, 1.3]) - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.04, 0.04, size=(inner.sum(), 3))
    return Mesh(v, mesh.elements)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [1, 2, 4, 7])
def test_constant_and_linear_fields_volume_term(dtype, n):
    mesh = _mesh(n)
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    nodes = map_nodes(mesh, elem)                           # (K, Np, 3)
    k, n_p = mesh.num_elements, elem.num_nodes
    # rounding scale of a derivative: |u| * max row sum |D| * max |dr/dx| (fp32 D has ~1e-7 row sums)
    dscale = np.abs(elem.diff).sum(axis=2).max() * np.abs(op.geometry.inv_jacobians).max()
    rel = {torch.float32: 1e-6, torch.float64: 1e-13}[dtype]
    const = np.ascontiguousarray(np.broadcast_to(np.arange(1.0, 7.0)[:, None, None], (6, k, n_p)))
    vol = op.from_padded(op.volume_padded(op.to_padded(const))).cpu().numpy()
    assert np.abs(vol).max() < rel * dscale * 6.0
    grad = np.random.default_rng(n).normal(size=(6, 3))     # u_c = grad[c] . x
    lin = np.einsum("cd,kpd->ckp", grad, nodes)
    vol = op.from_padded(op.volume_padded(op.to_padded(lin))).cpu().numpy()
    g = grad  # d u_c / d x_d = g[c, d]
    curl_e = np.array([g[2, 1] - g[1, 2], g[0, 2] - g[2, 0], g[1, 0] - g[0, 1]])
    curl_h = np.array([g[5, 1] - g[4, 2], g[3, 2] - g[5, 0], g[4, 0] - g[3, 1]])
    want = np.concatenate([curl_h, -curl_e])[:, None, None]  # vacuum: (curl H, -curl E)
    assert np.abs(vol - want).max() < rel * dscale * np.abs(lin).max()


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [1, 3, 5])
def test_continuous_linear_field_interior_fluxes_vanish(dtype, n):
    mesh = _mesh(10 + n)
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    grad = np.random.default_rng(20).normal(size=(6, 3))
    lin = np.einsum("cd,kpd->ckp", grad, map_nodes(mesh, elem))
    got = op.surface_flux(op.to_padded(lin)).cpu().numpy().reshape(6, mesh.num_elements, 4, -1)
    interior = ~op.is_boundary
    assert interior.sum() > 0
    assert np.abs(got[:, interior]).max() < TOL[dtype] * np.abs(lin).max()
    assert np.abs(got[:, ~interior]).max() > 1e-3  # PEC walls do see a jump


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("n", [2, 4])
def test_two_sided_flux_is_conservative(dtype, n):
    """minus-side + plus-side upwind brackets = n . (F(u-) - F(u+)) on every interior node pair."""
    mesh = _mesh(30 + n)
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    k, n_p, n_fp = mesh.num_elements, elem.num_nodes, elem.num_face_nodes
    u = np.random.default_rng(n).normal(size=(6, k, n_p))
    uq = op.from_padded(op.to_padded(u)).cpu().numpy()  # the values the kernel saw (fp32-rounded)
    br = op.surface_flux(op.to_padded(u)).cpu().numpy().reshape(6, k, 4, n_fp)
    br = br / op.geometry.face_jacobians[None, :, :, None]  # unscaled brackets
    flat = uq.reshape(6, -1)
    vm, vp = op.vmap_minus, op.vmap_plus
    nbr = op.maps.neighbors
    checked = 0
    for e in range(k):
        for f in range(4):
            if op.is_boundary[e, f]:
                continue
            e2 = int(nbr[e, f])
            f2 = int(np.nonzero(nbr[e2] == e)[0][0])
            # partner slot j of each node i: vmap_minus[e2, f2, j] == vmap_plus[e, f, i]
            j = np.argsort(vm[e2, f2])[np.searchsorted(np.sort(vm[e2, f2]), vp[e, f])]
            assert np.array_equal(vm[e2, f2, j], vp[e, f])
            um, up = flat[:, vm[e, f]], flat[:, vp[e, f]]
            df = flux(um) - flux(up)                       # (3, 6, Nfp)
            want = np.einsum("d,dcn->cn", op.normals[e, f], df)
            got = br[:, e, f, :] + br[:, e2, f2, j]
            assert np.abs(got - want).max() < 50 * TOL[dtype] * max(1.0, np.abs(want).max())
            checked += 1
    assert checked > 0
