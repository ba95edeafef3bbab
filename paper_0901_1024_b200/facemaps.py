"""Face-pair maps: the reference's vmaps and the compact device encoding.

The reference gathers traces through two int64 maps of shape (K, 4, Nfp),
``vmap_minus`` and ``vmap_plus``, built with a Python loop over interior faces
(oracle.py:110-127).  The stage kernel instead reads, per element face, one
neighbor id and one *code*: a row of a tiny table holding the neighbor's
node ids along the shared face (the row ``vmap_plus[k, f] - neighbor * Np``).
A box mesh needs 10 codes, any conforming mesh at most 4*4*6*2.  Per element
that is 8 int32 words instead of 8*Nfp int64 words.

``FaceMaps.vmap_plus`` rebuilds the reference map from the encoding, so the
bit-exact check against the reference's loop covers exactly what the kernel
reads.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import VERTEX_PERMUTATIONS, FaceConnectivity, Mesh, build_connectivity
from .refelem import NUM_FACES, ReferenceElement, face_node_permutation


@dataclass
class FaceMaps:
    num_nodes: int
    face_nodes: np.ndarray   # (4, Nfp) int64
    neighbors: np.ndarray    # (K, 4) int32, self for boundary faces
    codes: np.ndarray        # (K, 4) int32, -1 on PEC walls
    code_table: np.ndarray   # (num_codes, Nfp) uint8 node ids in the neighbor

    @property
    def num_elements(self) -> int:
        return len(self.neighbors)

    @property
    def is_boundary(self) -> np.ndarray:
        return self.codes < 0

    @property
    def vmap_minus(self) -> np.ndarray:
        k = np.arange(self.num_elements, dtype=np.int64)
        return k[:, None, None] * self.num_nodes + self.face_nodes[None, :, :]

    @property
    def vmap_plus(self) -> np.ndarray:
        vm = self.vmap_minus
        bnd = self.is_boundary
        codes = np.where(bnd, 0, self.codes)
        table = self.code_table.astype(np.int64) if len(self.code_table) else \
            np.zeros((1, self.face_nodes.shape[1]), dtype=np.int64)
        vp = self.neighbors.astype(np.int64)[:, :, None] * self.num_nodes + table[codes]
        return np.where(bnd[:, :, None], vm, vp)


def build_face_maps(mesh: Mesh, elem: ReferenceElement,
                    connectivity: FaceConnectivity | None = None) -> FaceMaps:
    """Vectorised equivalent of build_reference_operator's map loop (oracle.py:110-127)."""
    if connectivity is None:
        connectivity = build_connectivity(mesh)
    k_total, n_fp = mesh.num_elements, elem.num_face_nodes
    if elem.num_nodes > 256:
        raise ValueError("code tables store node ids as uint8")
    neighbors = np.repeat(np.arange(k_total, dtype=np.int32)[:, None], NUM_FACES, axis=1)
    codes = np.full((k_total, NUM_FACES), -1, dtype=np.int32)
    c = connectivity
    km, fm, kp, fp, pid = c.elem_minus, c.face_minus, c.elem_plus, c.face_plus, c.perm_id
    combo = (fm * NUM_FACES + fp) * len(VERTEX_PERMUTATIONS) + pid
    tables: dict = {}

    def code_of(row: np.ndarray) -> int:
        key = row.astype(np.uint8).tobytes()
        if key not in tables:
            tables[key] = len(tables)
        return tables[key]

    for cval in np.unique(combo):
        sel = combo == cval
        f_m, f_p, p = int(fm[sel][0]), int(fp[sel][0]), int(pid[sel][0])
        sigma = face_node_permutation(elem, f_m, f_p, VERTEX_PERMUTATIONS[p])
        minus_row = elem.face_nodes[f_p][sigma]            # vmap_plus[km, fm] - kp*Np
        plus_row = elem.face_nodes[f_m][np.argsort(sigma)]  # vmap_plus[kp, fp] - km*Np
        cm, cp = code_of(minus_row), code_of(plus_row)
        neighbors[km[sel], f_m] = kp[sel]
        codes[km[sel], f_m] = cm
        neighbors[kp[sel], f_p] = km[sel]
        codes[kp[sel], f_p] = cp
    # every boundary face is a PEC wall whatever its tag, as in face_states (oracle.py:56-57)
    table = np.zeros((len(tables), n_fp), dtype=np.uint8)
    for key, idx in tables.items():
        table[idx] = np.frombuffer(key, dtype=np.uint8)
    return FaceMaps(num_nodes=elem.num_nodes, face_nodes=np.asarray(elem.face_nodes, dtype=np.int64),
                    neighbors=neighbors, codes=codes, code_table=table)
