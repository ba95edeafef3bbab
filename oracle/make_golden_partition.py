"""Golden partitions of the reference's Alg. 2 (simtdg.layout.greedy_partition, layout.py:59-117).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_partition.py

Writes tests/golden/partition.npz: for a few meshes (the C1 box, a vertex-shuffled jittered box, a
two-component mesh) and block sizes, the reference's blocks as (element order, block offsets).
Build container only; the fixtures pin paper_0901_1024_b200.ordering.greedy_partition.
"""

from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "partition.npz")


def meshes():
    from simtdg.mesh import Mesh, generate_box_mesh

    yield "c1", generate_box_mesh((1.0, 1.0, 1.0), (6, 6, 7))
    rng = np.random.default_rng(5)
    box = generate_box_mesh((1.0, 1.0, 1.0), (5, 4, 3))
    v = box.vertices.copy()
    inner = np.all((v > 1e-9) & (v < 1 - 1e-9), axis=1)
    v[inner] += rng.uniform(-0.05, 0.05, size=(inner.sum(), 3))
    perm = rng.permutation(box.num_elements)
    yield "shuffled", Mesh(v, np.array([rng.permutation(r) for r in box.elements[perm]]))
    a = generate_box_mesh((1.0, 1.0, 1.0), (2, 2, 2))
    b = generate_box_mesh((1.0, 1.0, 1.0), (2, 1, 1))
    verts = np.concatenate([a.vertices, b.vertices + np.array([5.0, 0.0, 0.0])])
    elems = np.concatenate([a.elements, b.elements + len(a.vertices)])
    order = np.random.default_rng(9).permutation(len(elems))
    yield "two_components", Mesh(verts, elems[order])


def main() -> None:
    from simtdg.layout import greedy_partition
    from simtdg.mesh import build_connectivity

    out = {}
    for name, mesh in meshes():
        out[f"{name}_vertices"] = mesh.vertices
        out[f"{name}_elements"] = mesh.elements.astype(np.int32)
        conn = build_connectivity(mesh)
        for size in (1, 5, 16, 64):
            blocks = greedy_partition(mesh, size, conn)
            out[f"{name}_b{size}_order"] = np.concatenate([np.asarray(b, dtype=np.int32) for b in blocks])
            out[f"{name}_b{size}_offsets"] = np.cumsum([0] + [len(b) for b in blocks]).astype(np.int32)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
