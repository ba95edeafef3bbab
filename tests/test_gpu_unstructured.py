"""GPU parity on an unstructured (many-code) tetrahedral mesh read through the TetGen path.

A jittered 16x16x7 box (10,752 tets) whose elements list their vertices in random order is
written as TetGen .node/.ele text (1-based) and read back with read_tetgen, so faces glue through
many (f-, f+, permutation) combinations (reference mesh.py:147-228 and the
face_node_permutation tables, refelem.py:449-467) instead of the box's handful.  The fp32 tensor
path and the fp64 SIMT path are compared with the CPU oracle (reference algorithm) on the RHS of
a random state and on three LSRK4 steps of the cavity mode.
"""

import numpy as np
import pytest
from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import build_oracle_operator, rk4_step  # noqa: E402
from paper_0901_1024_b200 import (CavityMode, Mesh, build_b200_operator, build_reference_element,  # noqa: E402
                                  compute_geometry, generate_box_mesh, map_nodes, read_tetgen, stable_dt)


def _tetgen_text(mesh):
    node = [f"{len(mesh.vertices)} 3 0 0"] + [f"{i + 1} {float(x)!r} {float(y)!r} {float(z)!r}" for i, (x, y, z) in enumerate(mesh.vertices)]
    ele = [f"{len(mesh.elements)} 4 0"] + [f"{i + 1} " + " ".join(str(v + 1) for v in e)
                                           for i, e in enumerate(mesh.elements)]
    return "\n".join(node) + "\n", "\n".join(ele) + "\n"


@pytest.fixture(scope="module")
def mesh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    rng = np.random.default_rng(2024)
    box = generate_box_mesh((1.0, 1.0, 0.5), (16, 16, 7))
    v = box.vertices.copy()
    inner = np.all((v > 1e-9) & (v < np.array([1, 1, 0.5]) - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.012, 0.012, size=(inner.sum(), 3))
    shuffled = Mesh(v, np.array([rng.permutation(r) for r in box.elements]))
    return read_tetgen(*_tetgen_text(shuffled))


@pytest.mark.parametrize("order", [4, 6])
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.float64, 1e-12)])
def test_unstructured_rhs_and_steps(mesh, order, dtype, tol):
    assert mesh.num_elements >= 10_000
    elem = build_reference_element(order)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    ncodes = len(op.maps.code_table)
    assert ncodes > 20, f"only {ncodes} face codes"
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(order).normal(size=(6, mesh.num_elements, elem.num_nodes))
    err = rel_l2(op.rhs(state), ora.rhs(state))
    print(f"N={order} {dtype} codes={ncodes} path={op.path} rhs rel L2 {err:.2e}")
    assert err < (1e-13 if dtype == torch.float64 else tol)
    if order == 6 and dtype == torch.float64:
        return  # the oracle's N=6 steps on 10k tets take a minute; the RHS check above covers it
    u0 = CavityMode(1, 1, 1, (1.0, 1.0, 0.5)).evaluate(map_nodes(mesh, elem), 0.0)
    dt = stable_dt(mesh, compute_geometry(mesh), order)
    want = u0
    for _ in range(3):
        want = rk4_step(want, 0.0, dt, lambda t, y: ora.rhs(y))
    u = op.to_padded(u0)
    op.advance(u, dt, 3)
    err = rel_l2(op.from_padded(u).cpu().numpy(), want)
    print(f"N={order} {dtype} 3 steps rel L2 {err:.2e}")
    assert err < tol


@pytest.mark.parametrize("reorder", ["greedy", "morton", False])
def test_unstructured_orderings_match_oracle(mesh, reorder):
    """Internal element orders (the paper's Alg. 2 blocks, Morton, none) leave the natural-order
    results unchanged on the many-code mesh."""
    elem = build_reference_element(4)
    op = build_b200_operator(mesh, elem, reorder=reorder)
    ora = build_oracle_operator(mesh, elem)
    state = np.random.default_rng(3).normal(size=(6, mesh.num_elements, elem.num_nodes))
    assert rel_l2(op.rhs(state), ora.rhs(state)) < 1e-5
