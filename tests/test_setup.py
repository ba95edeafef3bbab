"""Host setup layer: reference element, mesh, connectivity, geometry, face maps.

Floats are pinned to the real reference's output (tests/golden); integer maps
must be bit-exact, against the golden arrays and against the oracle's
dict/loop restatement of the reference algorithm.
"""

import itertools

import numpy as np
import pytest
from conftest import golden_element, load_golden

from oracle import OracleOperator, oracle_sigma
from paper_0901_1024_b200 import refelem as R
from paper_0901_1024_b200.facemaps import build_face_maps
from paper_0901_1024_b200.maxwell import (VACUUM, CavityMode, Material, field_energy, pec_boundary,
                                          stable_dt, upwind_flux)
from paper_0901_1024_b200.mesh import (VERTEX_PERMUTATIONS, Mesh, NonConformingMeshError, build_connectivity,
                                       compute_geometry, generate_box_mesh, map_nodes, read_tetgen)
from paper_0901_1024_b200.stepper import rk4_step

DOF_TABLE = {1: (4, 3), 2: (10, 6), 3: (20, 10), 4: (35, 15), 5: (56, 21), 6: (84, 28), 7: (120, 36),
             8: (165, 45), 9: (220, 55)}


@pytest.mark.parametrize("order,expected", sorted(DOF_TABLE.items()))
def test_node_counts(order, expected):
    assert R.simplex_node_count(order) == expected


def test_bad_orders_rejected():
    with pytest.raises(ValueError):
        R.simplex_node_count(0)
    for bad in (0, 10):
        with pytest.raises(ValueError):
            R.build_reference_element(bad)


@pytest.mark.parametrize("n", range(1, 10))
def test_reference_element_matches_reference(golden_refelem, n):
    e = R.build_reference_element(n)
    g = golden_refelem
    assert np.array_equal(e.face_nodes, g[f"n{n}_face_nodes"].astype(np.int64))
    assert np.abs(e.nodes - g[f"n{n}_nodes"]).max() < 1e-14
    for name in ("diff", "lift", "mass", "face_mass", "face_barycentrics"):
        want = g[f"n{n}_{name}"]
        err = np.abs(getattr(e, name) - want).max() / np.abs(want).max()
        assert err < 1e-13, (name, err)
    assert not e.diff.flags.writeable


@pytest.mark.parametrize("n", [1, 3, 4, 6, 9])
def test_sigma_tables_match_oracle_restatement(golden_refelem, n):
    e = R.build_reference_element(n)
    gbar = golden_refelem[f"n{n}_face_barycentrics"]
    for fm, fp in itertools.product(range(4), range(4)):
        for p in VERTEX_PERMUTATIONS:
            assert np.array_equal(R.face_node_permutation(e, fm, fp, p), oracle_sigma(gbar, fm, fp, p))


def test_box_mesh_connectivity_geometry_match_reference_c1():
    g = load_golden("mesh_c1.npz")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (6, 6, 7))
    assert np.array_equal(mesh.vertices, g["vertices"])
    assert np.array_equal(mesh.elements, g["elements"])
    c = build_connectivity(mesh)
    got = np.stack([c.elem_minus, c.face_minus, c.elem_plus, c.face_plus, c.perm_id], axis=1)
    assert np.array_equal(got, g["interior"])
    assert np.array_equal(np.stack([c.bnd_elem, c.bnd_face, c.bnd_tag_id], axis=1), g["boundary"])
    assert c.tags == ("pec",)
    geo = compute_geometry(mesh)
    for name in ("inv_jacobians", "det_jacobians", "normals", "face_jacobians"):
        assert np.array_equal(getattr(geo, name), g[name]), name


def test_face_maps_bit_exact_vs_reference_c1():
    g = load_golden("mesh_c1.npz")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (6, 6, 7))
    fm = build_face_maps(mesh, R.build_reference_element(3))
    assert np.array_equal(fm.vmap_minus, g["vmap_minus"])
    assert np.array_equal(fm.vmap_plus, g["vmap_plus"])
    assert np.array_equal(fm.is_boundary, g["is_boundary"])


def _jittered_tet_mesh(seed):
    """A box mesh with jittered interior vertices and shuffled local vertex order.

    Shuffling exercises many (face-, face+, perm) combinations -- the box mesh
    alone only produces 5 of the 96 possible ones.
    """
    rng = np.random.default_rng(seed)
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (2, 2, 2))
    v = mesh.vertices.copy()
    interior = np.all((v > 1e-9) & (v < 1 - 1e-9), axis=1)
    v[interior] += rng.uniform(-0.08, 0.08, size=(interior.sum(), 3))
    e = np.array([rng.permutation(row) for row in mesh.elements])
    return Mesh(v, e)


@pytest.mark.parametrize("n", [1, 2, 4, 7])
@pytest.mark.parametrize("seed", [0, 1])
def test_face_maps_bit_exact_vs_oracle_shuffled(golden_refelem, n, seed):
    mesh = _jittered_tet_mesh(seed)
    fm = build_face_maps(mesh, R.build_reference_element(n))
    ora = OracleOperator(mesh.vertices, mesh.elements, golden_element(golden_refelem, n))
    assert np.array_equal(fm.vmap_minus, ora.vmap_minus)
    assert np.array_equal(fm.vmap_plus, ora.vmap_plus)
    assert np.array_equal(fm.is_boundary, ora.is_boundary)
    c = build_connectivity(mesh)
    got = np.stack([c.elem_minus, c.face_minus, c.elem_plus, c.face_plus, c.perm_id], axis=1)
    assert np.array_equal(got, ora.interior)
    assert len(np.unique(c.face_minus * 24 + c.face_plus * 6 + c.perm_id)) > 5


def test_permuted_face_nodes_coincide():
    mesh = _jittered_tet_mesh(3)
    elem = R.build_reference_element(3)
    fm = build_face_maps(mesh, elem)
    x = map_nodes(mesh, elem).reshape(-1, 3)
    inner = ~fm.is_boundary
    assert np.abs(x[fm.vmap_minus[inner]] - x[fm.vmap_plus[inner]]).max() < 1e-10


def test_connectivity_identities_and_errors():
    for cells in [(1, 1, 1), (2, 2, 1), (2, 2, 2), (3, 1, 2)]:
        mesh = generate_box_mesh((1, 1, 1), cells)
        c = build_connectivity(mesh)
        assert 4 * mesh.num_elements == 2 * c.num_interior + c.num_boundary
        nx, ny, nz = cells
        assert c.num_boundary == 4 * (nx * ny + ny * nz + nx * nz)
    verts = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1]])
    with pytest.raises(NonConformingMeshError):
        build_connectivity(Mesh(verts, np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]])))
    with pytest.raises(ValueError):
        generate_box_mesh((1, 0, 1), (1, 1, 1))
    with pytest.raises(ValueError):
        generate_box_mesh((1, 1, 1), (1, 0, 1))
    with pytest.raises(ValueError):
        compute_geometry(Mesh(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0.5, 0.5, 0]]),
                              np.array([[0, 1, 2, 3]])))


def test_orientation_repair_and_tetgen():
    node = "4 3 0 0\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n"
    mesh = read_tetgen(node, "1 4 0\n1 1 3 2 4\n")
    assert (mesh.element_volumes() > 0).all()
    c = build_connectivity(mesh)
    assert c.num_interior == 0 and c.num_boundary == 4


def test_boundary_tags_numbered_by_first_appearance():
    mesh = generate_box_mesh((1, 1, 1), (1, 1, 1))
    c0 = build_connectivity(mesh)
    k, f = int(c0.bnd_elem[3]), int(c0.bnd_face[3])
    key = tuple(sorted(mesh.face_vertex_triple(k, f)))
    mesh.boundary_tags = {key: "port"}
    c = build_connectivity(mesh)
    assert c.tags == ("pec", "port")
    assert int(c.bnd_tag_id[3]) == 1 and int(c.bnd_tag_id.sum()) == 1


def test_flux_known_answers():
    g = load_golden("flux_known.npz")
    assert np.allclose(upwind_flux(g["um"], g["up"], g["normal"]), g["bracket"], atol=1e-15)
    rng = np.random.default_rng(1)
    u = rng.normal(size=6)
    n = np.array([0.0, 0.6, 0.8])
    assert np.allclose(upwind_flux(u, u, n), 0.0, atol=1e-15)
    assert np.allclose(pec_boundary(pec_boundary(u, n), n), u, atol=1e-15)
    with pytest.raises(ValueError):
        Material(permittivity=0.0)


def test_stable_dt_c1_and_cavity():
    g = load_golden("c1_n3.npz")
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (6, 6, 7))
    assert stable_dt(mesh, compute_geometry(mesh), 3) == float(g["dt"])
    with pytest.raises(ValueError):
        stable_dt(mesh, compute_geometry(mesh), 3, cfl=0.0)
    elem = R.build_reference_element(3)
    u0 = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0)
    assert np.abs(u0[3:]).max() == 0.0
    assert field_energy(u0, elem, compute_geometry(mesh), VACUUM) == pytest.approx(float(g["energies"][0]),
                                                                                   rel=1e-13)


class TestRk4:
    def test_zero_rhs_keeps_state(self):
        y = np.array([1.0, -2.0, 3.0])
        assert np.array_equal(rk4_step(y, 0.0, 0.1, lambda t, u: np.zeros_like(u)), y)

    def test_fourth_order_ratio(self):
        lam = -1.3

        def err(dt):
            return abs(float(rk4_step(np.array(1.0), 0.0, dt, lambda t, u: lam * u)) - np.exp(lam * dt))

        assert err(0.1) / err(0.05) == pytest.approx(32.0, rel=0.10)

    def test_torch_path_matches_numpy(self):
        torch = pytest.importorskip("torch")
        rng = np.random.default_rng(15)
        a = rng.normal(size=(4, 4))
        y0 = rng.normal(size=4)
        want = rk4_step(y0, 0.0, 0.05, lambda t, u: a @ u)
        ta = torch.tensor(a)
        got = rk4_step(torch.tensor(y0), 0.0, 0.05, lambda t, u: ta @ u)
        assert np.abs(got.numpy() - want).max() < 1e-14

    def test_rejects_bad_dt(self):
        with pytest.raises(ValueError):
            rk4_step(np.zeros(2), 0.0, 0.0, lambda t, u: u)


def test_cli_error_boundary_and_eoc_fit(capsys):
    """JSON error on stderr + rc 1 at the process boundary (reference cli.py:408-411)."""
    import json

    from paper_0901_1024_b200.cli import fit_eoc, main, rows_to_csv

    assert main(["simulate", "--node-file", "only-one.node"]) == 1
    err = json.loads(capsys.readouterr().err.strip().splitlines()[-1])
    assert set(err) == {"error", "message"}
    h = np.array([0.5, 0.25, 0.125])
    assert abs(fit_eoc(h, 3.0 * h ** 4.2) - 4.2) < 1e-12
    assert rows_to_csv([{"a": 0.1, "b": 2}]) == "a,b\n0.10000000000000001,2\n"


def test_morton_order_and_map_relabelling():
    """Internal locality order (ordering.py): a permutation, tiles are compact, maps relabelled consistently."""
    from paper_0901_1024_b200.facemaps import build_face_maps
    from paper_0901_1024_b200.ordering import column_order, morton_order, permute_maps

    mesh = generate_box_mesh((1.0, 1.0, 1.0), (12, 12, 12))
    elem = R.build_reference_element(2)
    order = morton_order(mesh.vertices, mesh.elements)
    k = mesh.num_elements
    assert np.array_equal(np.sort(order), np.arange(k))
    maps = build_face_maps(mesh, elem)
    pm = permute_maps(maps, order)
    inner = pm.codes >= 0
    assert np.array_equal(order[pm.neighbors[inner]], maps.neighbors[order][inner])
    assert np.array_equal(pm.codes, maps.codes[order])
    # 64-element tiles: more face neighbours inside the tile than with the reference numbering
    def in_tile(nbr, codes):
        idx = np.arange(len(nbr))[:, None] // 64
        m = codes >= 0
        return float(((nbr // 64) == idx)[m].mean())
    assert in_tile(pm.neighbors, pm.codes) > in_tile(maps.neighbors, maps.codes)
    col = column_order(mesh.vertices, mesh.elements)
    assert np.array_equal(np.sort(col), np.arange(k))
    pc = permute_maps(maps, col)
    assert in_tile(pc.neighbors, pc.codes) > in_tile(maps.neighbors, maps.codes)


@pytest.mark.parametrize("order", [2, 4, 9])
def test_face_slot_order_and_code_tables(order):
    """Face-node slot order (ordering.face_slot_order): a per-face permutation that lowers the modelled
    shared-bank cost, and permute_face_slots keeps every (face node -> neighbour node) pairing."""
    from paper_0901_1024_b200.ordering import (_bank_cost, _flux_lane_groups, face_slot_order,
                                               permute_face_slots)

    elem = R.build_reference_element(order)
    fm = np.asarray(elem.face_nodes)
    nfp = fm.shape[1]
    npg, nfpk = (elem.num_nodes + 3) // 4 * 4, (nfp + 7) // 8 * 8
    perm = face_slot_order(fm, order, npg, nfpk)
    base, slots, live = _flux_lane_groups(order, npg, nfp, nfpk)
    for f in range(4):
        assert np.array_equal(np.sort(perm[f]), np.arange(nfp))
        assert _bank_cost(fm[f][perm[f]], base, slots, live) <= _bank_cost(fm[f], base, slots, live)
    if order == 4:  # 2-way conflicts of the natural order removed on average
        assert np.mean([_bank_cost(fm[f][perm[f]], base, slots, live) for f in range(4)]) < 1.2 * len(base)
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (3, 2, 2))
    maps = build_face_maps(mesh, elem)
    pm = permute_face_slots(maps, perm)
    assert np.array_equal(pm.neighbors, maps.neighbors)
    assert np.array_equal(pm.codes >= 0, maps.codes >= 0)
    for f in range(4):
        assert np.array_equal(pm.face_nodes[f], fm[f][perm[f]])
        inner = maps.codes[:, f] >= 0
        got = pm.code_table[pm.codes[inner, f]]                  # slot i -> neighbour node
        want = maps.code_table[maps.codes[inner, f]][:, perm[f]]  # natural node perm[f, i]
        assert np.array_equal(got, want)


def test_tetgen_roundtrip_and_errors():
    """read_tetgen: 0/1-based numbering, shuffled record order, bytes, comments, malformed input."""
    from paper_0901_1024_b200 import MeshFormatError

    mesh = generate_box_mesh((1.0, 2.0, 1.0), (2, 1, 2))
    rng = np.random.default_rng(1)
    for base in (0, 1):
        # the numbering base is read from the first point record (reference behaviour), so it stays first
        pord = np.concatenate([[0], 1 + rng.permutation(len(mesh.vertices) - 1)])
        eord = rng.permutation(mesh.num_elements)
        node = f"# comment\n{len(mesh.vertices)} 3 0 0\n" + "".join(
            f"{i + base} {float(x)!r} {float(y)!r} {float(z)!r}  # pt\n" for i, (x, y, z) in zip(pord, mesh.vertices[pord]))
        ele = f"{mesh.num_elements} 4 0\n" + "".join(
            f"{i + base} " + " ".join(str(v + base) for v in mesh.elements[i]) + "\n" for i in eord)
        got = read_tetgen(node.encode(), ele)
        assert np.array_equal(got.vertices, mesh.vertices) and np.array_equal(got.elements, mesh.elements)
    bad = [("4 3\n1 0 0 0\n2 1 0 0\n3 0 1 0\n", "1 4\n1 1 2 3 4\n"),          # fewer points than announced
           ("4 3\n1 0 0 0\n1 1 0 0\n3 0 1 0\n4 0 0 1\n", "1 4\n1 1 2 3 4\n"),  # duplicate point id
           ("4 3\n2 0 0 0\n3 1 0 0\n4 0 1 0\n5 0 0 1\n", "1 4\n2 2 3 4 5\n"),  # numbering starts at 2
           ("4 3\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 z\n", "1 4\n1 1 2 3 4\n"),  # non-numeric coordinate
           ("4 3\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n", "1 4\n1 1 2 3\n"),    # short element record
           ("4 3\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n", "")]                  # empty .ele
    for node, ele in bad:
        with pytest.raises(MeshFormatError):
            read_tetgen(node, ele)


def test_greedy_partition_matches_reference_golden():
    """ordering.greedy_partition == the reference's Alg. 2 (layout.py:59-117) block for block: golden
    partitions made by simtdg itself (oracle/make_golden_partition.py), incl. a vertex-shuffled mesh
    and a two-component mesh (reseeding)."""
    from paper_0901_1024_b200.ordering import greedy_block_order, greedy_partition

    g = load_golden("partition.npz")
    for name in ("c1", "shuffled", "two_components"):
        mesh = Mesh(g[f"{name}_vertices"], g[f"{name}_elements"].astype(np.int64))
        conn = build_connectivity(mesh)
        for size in (1, 5, 16, 64):
            blocks = greedy_partition(mesh, size, conn)
            assert np.array_equal(np.concatenate(blocks), g[f"{name}_b{size}_order"])
            assert np.array_equal(np.cumsum([0] + [len(b) for b in blocks]), g[f"{name}_b{size}_offsets"])
            assert all(1 <= len(b) <= size for b in blocks)
        order = greedy_block_order(mesh.vertices, mesh.elements, 16, conn)
        assert np.array_equal(np.sort(order), np.arange(mesh.num_elements))
    with pytest.raises(ValueError):
        greedy_partition(generate_box_mesh((1.0, 1.0, 1.0), (1, 1, 1)), 0)
