"""Generate tests/golden/*.npz from the REAL reference package (build container only).

Run from the repo root:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

It imports simtdg from the read-only reference tree, evaluates the hot path on
small seeded inputs and stores inputs + outputs.  The fixtures pin
(a) the oracle restatement (tests/test_oracle_golden.py) and (b) the product's
host setup (refelem / mesh / maps) and, through the GPU tests, the kernels.
/root/reference is not needed afterwards (it does not exist on the GPU box).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def main() -> None:
    from simtdg.kernels import build_reference_operator, gather_stage, rk4_step
    from simtdg.maxwell import CavityMode, field_energy, stable_dt, upwind_flux
    from simtdg.mesh import Mesh, build_connectivity, compute_geometry, generate_box_mesh, map_nodes
    from simtdg.refelem import build_reference_element

    os.makedirs(OUT, exist_ok=True)

    # 1. reference elements N = 1..9
    ref = {}
    for n in range(1, 10):
        e = build_reference_element(n)
        for name in ("nodes", "diff", "lift", "mass", "face_mass", "face_barycentrics"):
            ref[f"n{n}_{name}"] = np.asarray(getattr(e, name))
        ref[f"n{n}_face_nodes"] = np.asarray(e.face_nodes).astype(np.int16)
    np.savez_compressed(os.path.join(OUT, "refelem.npz"), **ref)

    # 2. C1 mesh: connectivity, geometry, N=3 index maps
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (6, 6, 7))
    conn = build_connectivity(mesh)
    geo = compute_geometry(mesh)
    op = build_reference_operator(mesh, build_reference_element(3), connectivity=conn)
    np.savez_compressed(
        os.path.join(OUT, "mesh_c1.npz"),
        vertices=mesh.vertices, elements=mesh.elements.astype(np.int32),
        interior=np.stack([conn.elem_minus, conn.face_minus, conn.elem_plus, conn.face_plus,
                           conn.perm_id], axis=1).astype(np.int32),
        boundary=np.stack([conn.bnd_elem, conn.bnd_face, conn.bnd_tag_id], axis=1).astype(np.int32),
        inv_jacobians=geo.inv_jacobians, det_jacobians=geo.det_jacobians, normals=geo.normals,
        face_jacobians=geo.face_jacobians,
        vmap_minus=op.vmap_minus.astype(np.int32), vmap_plus=op.vmap_plus.astype(np.int32),
        is_boundary=op.is_boundary)

    # 3. RHS / flux on small meshes, N = 1..6 (and a single N=7 / N=9 tet)
    small = {}
    rng_seed = 12
    for n in range(1, 7):
        m = generate_box_mesh((1.0, 0.9, 1.1), (1, 2, 1))
        e = build_reference_element(n)
        o = build_reference_operator(m, e)
        state = np.random.default_rng(rng_seed + n).normal(size=(6, m.num_elements, e.num_nodes))
        small[f"n{n}_state"] = state
        small[f"n{n}_rhs"] = o.rhs(state)
        small[f"n{n}_gather"] = gather_stage(o, state)
    tet = Mesh(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]]), np.array([[0, 1, 2, 3]]))
    for n in (7, 9):
        e = build_reference_element(n)
        o = build_reference_operator(tet, e)
        state = np.random.default_rng(21).normal(size=(6, 1, e.num_nodes))
        small[f"tet{n}_state"] = state
        small[f"tet{n}_rhs"] = o.rhs(state)
    np.savez_compressed(os.path.join(OUT, "rhs_small.npz"), **small)

    # 4. C1 headline case: N=3, cavity (1,1,1), 10 LSRK4 steps; plus a random-state RHS
    e3 = build_reference_element(3)
    mode = CavityMode(1, 1, 1, (1.0, 1.0, 1.0))
    u0 = mode.evaluate(map_nodes(mesh, e3), 0.0)
    dt = stable_dt(mesh, geo, 3, cfl=1.0)
    u = u0
    energies = [field_energy(u, e3, geo)]
    for _ in range(10):
        u = rk4_step(u, 0.0, dt, lambda t, y: op.rhs(y))
        energies.append(field_energy(u, e3, geo))
    rnd = np.random.default_rng(0).normal(size=u0.shape)
    np.savez_compressed(os.path.join(OUT, "c1_n3.npz"), dt=dt, u10=u, energies=np.array(energies),
                        rhs_random=op.rhs(rnd))

    # 5. N=4 on a (3,3,3) box: 10 steps from the cavity mode (the bench order)
    m4 = generate_box_mesh((1.0, 1.0, 1.0), (3, 3, 3))
    e4 = build_reference_element(4)
    g4 = compute_geometry(m4)
    o4 = build_reference_operator(m4, e4)
    u = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(m4, e4), 0.0)
    dt4 = stable_dt(m4, g4, 4, cfl=1.0)
    for _ in range(10):
        u = rk4_step(u, 0.0, dt4, lambda t, y: o4.rhs(y))
    np.savez_compressed(os.path.join(OUT, "box3_n4.npz"), dt=dt4, u10=u)

    # 6. known answers for the flux
    n = np.array([1.0, 0.0, 0.0])
    um = np.zeros(6)
    up = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 1.0])  # test_maxwell.py:86-92 frozen jump
    np.savez_compressed(os.path.join(OUT, "flux_known.npz"), normal=n, um=um, up=up,
                        bracket=upwind_flux(um, up, n))
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    sys.exit(main())
