"""Integer setup at benchmark scale: connectivity and face maps bit-exact against the oracle's
dict / loop restatement of the reference algorithm (mesh.py:263-300, oracle.py:110-127).

48k tets (C2's mesh) runs in the default CPU suite; 998,250 tets (C3, the headline mesh) is
marked slow and runs when DGM_SLOW=1 (several minutes of single-threaded Python in the oracle;
the committed log is profiles/r02/setup_scale_c3.log).
"""

import os

import numpy as np
import pytest

from oracle import oracle_connectivity, oracle_sigma
from oracle.dg_oracle import PERMS
from paper_0901_1024_b200 import build_reference_element, generate_box_mesh
from paper_0901_1024_b200.facemaps import build_face_maps
from paper_0901_1024_b200.mesh import build_connectivity


def _oracle_vmaps(interior, k_total, elem):
    """The reference's per-interior-face vmap loop (oracle.py:110-127), restated in the oracle."""
    n_p = elem.num_nodes
    fnodes = np.asarray(elem.face_nodes)
    vm = np.arange(k_total)[:, None, None] * n_p + fnodes[None, :, :]
    vp = vm.copy()
    cache = {}
    bary = np.asarray(elem.face_barycentrics)
    for km, fm, kp, fp, pid in interior.tolist():
        key = (fm, fp, pid)
        if key not in cache:
            cache[key] = oracle_sigma(bary, fm, fp, PERMS[pid])
        sigma = cache[key]
        vp[km, fm] = kp * n_p + fnodes[fp][sigma]
        vp[kp, fp] = km * n_p + fnodes[fm][np.argsort(sigma)]
    return vm, vp


def _check(cells, order):
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    interior, boundary = oracle_connectivity(mesh.elements)
    c = build_connectivity(mesh)
    got = np.stack([c.elem_minus, c.face_minus, c.elem_plus, c.face_plus, c.perm_id], axis=1)
    assert np.array_equal(got, interior)
    assert np.array_equal(np.stack([c.bnd_elem, c.bnd_face], axis=1), boundary)
    elem = build_reference_element(order)
    fm = build_face_maps(mesh, elem, c)
    vm, vp = _oracle_vmaps(interior, mesh.num_elements, elem)
    assert np.array_equal(fm.vmap_minus, vm)
    assert np.array_equal(fm.vmap_plus, vp)
    bnd = np.zeros((mesh.num_elements, 4), dtype=bool)
    bnd[boundary[:, 0], boundary[:, 1]] = True
    assert np.array_equal(fm.is_boundary, bnd)
    return mesh.num_elements


def test_connectivity_and_maps_bit_exact_c2_48k():
    assert _check((20, 20, 20), 4) == 48000


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("DGM_SLOW") != "1", reason="slow (minutes): set DGM_SLOW=1")
def test_connectivity_and_maps_bit_exact_c3_998k():
    assert _check((55, 55, 55), 4) == 998250
