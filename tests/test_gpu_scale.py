"""Parity at the benchmark sizes (BASELINE configs C3, C4, C5) -- the meshes the headline runs on.

Two independent checks per config:
  * sampled RHS: ~2,000 random elements of the full mesh; the oracle (reference algorithm,
    oracle.py:60-94) evaluates the RHS on the sub-mesh made of those elements plus all their
    face neighbours, so every sampled row sees exactly its true neighbourhood; the GPU's rows of
    the full-mesh RHS must match (fp32 <= 1e-5, fp64 <= 1e-12 relative L2 over the sampled rows);
  * 10 LSRK4 steps of the fp32 tensor-core path against the fp64 path (itself oracle-pinned on
    every small mesh) on the full mesh: relative L2 <= 1e-5 (BASELINE north_star tolerance).
The int64 element-row arithmetic (6 * 36 * 8M words per field slab at C4) is exercised here only.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import build_oracle_operator  # noqa: E402
from paper_0901_1024_b200 import (CavityMode, Mesh, build_b200_operator, build_connectivity,  # noqa: E402
                                  build_reference_element, generate_box_mesh, map_nodes, stable_dt)

CONFIGS = {  # name: (cells, order)
    "C3": ((55, 55, 55), 4),
    "C5": ((70, 70, 70), 6),
    "C4": ((110, 110, 110), 4),
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _dev_rel_l2(a: torch.Tensor, b: torch.Tensor) -> float:
    return float(torch.linalg.vector_norm((a - b).double()) / torch.linalg.vector_norm(b.double()))


def _sampled_rhs_error(mesh, elem, op, seed, nsample=2000):
    k = mesh.num_elements
    rng = np.random.default_rng(seed)
    sample = np.sort(rng.choice(k, nsample, replace=False))
    nbrs = op.maps.neighbors[sample]          # natural numbering; walls point at the element itself
    sub_ids = np.unique(np.concatenate([sample, nbrs.ravel().astype(np.int64)]))
    gen = torch.Generator(device="cuda").manual_seed(seed)
    state = torch.randn((6, k, elem.num_nodes), generator=gen, device="cuda", dtype=torch.float64)
    rows = op.from_padded(op.rhs_padded(op.to_padded(state)))
    got = rows[:, torch.as_tensor(sample, device="cuda")].cpu().numpy()
    ora = build_oracle_operator(Mesh(mesh.vertices, mesh.elements[sub_ids]), elem)
    want = ora.rhs(state[:, torch.as_tensor(sub_ids, device="cuda")].cpu().numpy())
    want = want[:, np.searchsorted(sub_ids, sample)]
    return float(np.linalg.norm(got - want) / np.linalg.norm(want)), len(sub_ids)


@pytest.fixture(scope="module")
def built():
    cache = {}

    def get(name):
        if name not in cache:
            cache.clear()  # one config resident at a time
            torch.cuda.empty_cache()
            cells, n = CONFIGS[name]
            mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
            cache[name] = (mesh, build_reference_element(n), build_connectivity(mesh))
        return cache[name]

    return get


@pytest.mark.parametrize("name", ["C3", "C5", "C4"])
def test_sampled_rhs_vs_oracle_at_scale(built, name):
    mesh, elem, conn = built(name)
    for dtype, tol in ((torch.float32, 1e-5), (torch.float64, 1e-12)):
        if name == "C4" and dtype == torch.float64:
            continue  # C4 is the fp32 strong-scaling config; fp64 runs on C3 / C5
        op = build_b200_operator(mesh, elem, connectivity=conn, dtype=dtype)
        if dtype == torch.float32:
            assert op.path == "tensor"
        err, nsub = _sampled_rhs_error(mesh, elem, op, seed=7)
        print(f"{name} {dtype} K={mesh.num_elements} sampled RHS rel L2 {err:.3e} (oracle sub-mesh {nsub} tets)")
        assert err < tol
        del op
        torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["C3", "C5", "C4"])
def test_ten_steps_fp32_tensor_vs_fp64_at_scale(built, name):
    mesh, elem, conn = built(name)
    nodes = map_nodes(mesh, elem)
    u0 = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(nodes, 0.0)
    del nodes
    ops = {}
    out = {}
    for dtype in (torch.float32, torch.float64):
        op = build_b200_operator(mesh, elem, connectivity=conn, dtype=dtype)
        dt = stable_dt(mesh, op.geometry, elem.order)
        u = op.to_padded(u0)
        e0 = op.field_energy(u)
        op.advance(u, dt, 10)
        e1 = op.field_energy(u)
        assert np.isfinite(e1) and e1 <= e0 * (1 + 1e-6)       # upwind DG dissipates energy
        assert op.check_padding(u)
        out[dtype] = op.from_padded(u, torch.float32 if dtype == torch.float32 else torch.float64)
        ops[dtype] = op.path
        del op, u
        torch.cuda.empty_cache()
    err = _dev_rel_l2(out[torch.float32], out[torch.float64])
    print(f"{name} K={mesh.num_elements} N={elem.order}: 10 steps {ops[torch.float32]} fp32 vs "
          f"{ops[torch.float64]} fp64 rel L2 {err:.3e}")
    assert ops[torch.float32] == "tensor"
    assert err < 1e-5


def test_sampled_rhs_unstructured_at_scale():
    """A 192,000-tet mesh with unstructured numbering (jittered vertices, every element's vertex list
    and the element order shuffled: many (f-, f+, perm) codes, no box locality) under the paper's
    Alg. 2 element order: sampled RHS rows vs the oracle, fp32 tensor path and fp64."""
    rng = np.random.default_rng(7)
    box = generate_box_mesh((1.0, 1.0, 0.5), (40, 40, 20))
    v = box.vertices.copy()
    inner = np.all((v > 1e-9) & (v < np.array([1.0, 1.0, 0.5]) - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.005, 0.005, size=(inner.sum(), 3))
    perm = rng.permutation(box.num_elements)
    mesh = Mesh(v, np.array([rng.permutation(r) for r in box.elements[perm]]))
    elem = build_reference_element(4)
    conn = build_connectivity(mesh)
    for dtype, tol in ((torch.float32, 1e-5), (torch.float64, 1e-12)):
        op = build_b200_operator(mesh, elem, connectivity=conn, dtype=dtype, reorder="greedy")
        assert len(op.maps.code_table) > 20
        err, nsub = _sampled_rhs_error(mesh, elem, op, seed=11)
        print(f"unstructured {dtype} K={mesh.num_elements} codes={len(op.maps.code_table)} path={op.path} "
              f"sampled RHS rel L2 {err:.3e}")
        assert err < tol
        del op
        torch.cuda.empty_cache()
