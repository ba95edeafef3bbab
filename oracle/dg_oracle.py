"""Numpy restatement of the reference DG Maxwell operator (TEST INFRASTRUCTURE).

Every function cites the reference code it restates (paths relative to
/root/reference/pkg/src/simtdg).  The restatement deliberately keeps the
reference's *algorithm* -- dict-based face matching, per-face loop for the
plus-side index map, einsum contractions, numpy elementwise flux -- so that it
is an independent check of the vectorised setup and of the CUDA kernels.  It
takes the mesh (vertices, elements) and a reference element (nodes, diff,
lift, face_nodes, face_barycentrics), both pinned to the real reference by
tests/golden (see make_golden.py).
"""

from __future__ import annotations

import itertools
import math

import numpy as np

FACE_VERTEX_IDS = ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3))            # refelem.py:34
FACE_AREAS = np.array([2.0, 2.0, 2.0 * math.sqrt(3.0), 2.0])             # refelem.py:49
_S3 = 1.0 / math.sqrt(3.0)
FACE_UNIT_NORMALS = np.array([[0, 0, -1.0], [0, -1.0, 0], [_S3, _S3, _S3], [-1.0, 0, 0]])  # refelem.py:39-46
PERMS = tuple(itertools.permutations(range(3)))                           # mesh.py:20

# assemble.py:80-102
RK_A = (0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
        -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0)
RK_B = (1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
        1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
        2277821191437.0 / 14882151754819.0)
RK_C = (0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
        2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0)


# ---------------------------------------------------------------------------
# setup: connectivity, sigma, geometry, index maps


def oracle_connectivity(elements: np.ndarray):
    """Face matching by dict on sorted vertex triples (mesh.py:263-300).

    Returns (interior (P,5) [km, fm, kp, fp, perm_id], boundary (B,2) [k, f]).
    """
    table: dict = {}
    for k in range(len(elements)):
        ids = elements[k]
        for f, corners in enumerate(FACE_VERTEX_IDS):
            tri = tuple(int(ids[c]) for c in corners)
            table.setdefault(tuple(sorted(tri)), []).append((k, f, tri))
    interior, boundary = [], []
    for key, owners in table.items():
        if len(owners) > 2:
            raise ValueError(f"non-conforming face {key}")
        if len(owners) == 2:
            (km, fm, tm), (kp, fp, tp) = sorted(owners)
            interior.append((km, fm, kp, fp, PERMS.index(tuple(tp.index(v) for v in tm))))
        else:
            boundary.append(owners[0][:2])
    interior.sort()
    boundary.sort()
    return np.array(interior, dtype=np.int64).reshape(-1, 5), np.array(boundary, dtype=np.int64).reshape(-1, 2)


def oracle_sigma(face_barycentrics: np.ndarray, fm: int, fp: int, perm) -> np.ndarray:
    """Glued-face node pairing via barycentrics rounded to 9 digits (refelem.py:449-467)."""
    minus = np.round(face_barycentrics[fm], 9)
    plus = np.round(face_barycentrics[fp], 9)
    where = {}
    for j in range(len(plus)):
        where[tuple(plus[j, list(perm)])] = j
    return np.array([where[tuple(minus[i])] for i in range(len(minus))], dtype=np.int64)


def oracle_geometry(vertices: np.ndarray, elements: np.ndarray) -> dict:
    """Affine factors (mesh.py:316-350)."""
    v, e = vertices, elements
    dxdr = np.empty((len(e), 3, 3))
    for mu in range(3):
        dxdr[:, :, mu] = (v[e[:, mu + 1]] - v[e[:, 0]]) / 2.0
    det = np.linalg.det(dxdr)
    drdx = np.linalg.inv(dxdr)
    nrm = np.einsum("fm,kmn->kfn", FACE_UNIT_NORMALS, drdx)
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    sj = np.empty((len(e), 4))
    for f, (a, b, c) in enumerate(FACE_VERTEX_IDS):
        pa, pb, pc = v[e[:, a]], v[e[:, b]], v[e[:, c]]
        sj[:, f] = 0.5 * np.linalg.norm(np.cross(pb - pa, pc - pa), axis=1) / FACE_AREAS[f]
    return {"dxdr": dxdr, "det": det, "drdx": drdx, "normals": nrm, "sj": sj}


# ---------------------------------------------------------------------------
# flux arithmetic


def pec_mirror(um: np.ndarray, n) -> np.ndarray:
    """E+ = -E- + 2(n.E-)n, H+ = H- - 2(n.H-)n   (maxwell.py:117-132)."""
    ndote = n[0] * um[0] + n[1] * um[1] + n[2] * um[2]
    ndoth = n[0] * um[3] + n[1] * um[4] + n[2] * um[5]
    out = np.empty_like(um)
    for c in range(3):
        out[c] = -um[c] + 2.0 * ndote * n[c]
        out[3 + c] = um[3 + c] - 2.0 * ndoth * n[c]
    return out


def _cross(a, b):
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def upwind_bracket(um: np.ndarray, up: np.ndarray, n, z: float = 1.0, y: float = 1.0) -> np.ndarray:
    """Uniform-material upwind bracket (maxwell.py:73-114 with Z+ = Z- = z)."""
    de = [up[c] - um[c] for c in range(3)]
    dh = [up[3 + c] - um[3 + c] for c in range(3)]
    nde, ndh = _cross(n, de), _cross(n, dh)
    ea = _cross(n, [z * dh[c] - nde[c] for c in range(3)])
    ha = _cross(n, [-y * de[c] - ndh[c] for c in range(3)])
    out = np.empty(np.broadcast_shapes(np.shape(um), np.shape(up)))
    for c in range(3):
        out[c] = ea[c] / (2.0 * z)
        out[3 + c] = ha[c] / (2.0 * y)
    return out


# ---------------------------------------------------------------------------
# operator


class OracleOperator:
    """Restates ReferenceMaxwellOperator (oracle.py:36-94)."""

    def __init__(self, vertices, elements, elem, eps: float = 1.0, mu: float = 1.0):
        self.elem = elem
        self.eps, self.mu = float(eps), float(mu)
        self.z = math.sqrt(self.mu / self.eps)
        self.y = 1.0 / self.z
        e = np.asarray(elements, dtype=np.int64)
        self.num_elements = len(e)
        self.geo = oracle_geometry(np.asarray(vertices, dtype=np.float64), e)
        self.interior, self.boundary = oracle_connectivity(e)
        k_total, n_p, n_fp = len(e), elem.num_nodes, elem.num_face_nodes
        fnodes = np.asarray(elem.face_nodes)
        # oracle.py:110-127 -- per-face loop over interior pairs
        vmap_minus = np.empty((k_total, 4, n_fp), dtype=np.int64)
        for f in range(4):
            vmap_minus[:, f, :] = np.arange(k_total)[:, None] * n_p + fnodes[f][None, :]
        vmap_plus = vmap_minus.copy()
        sig_cache: dict = {}
        for km, fm, kp, fp, pid in self.interior:
            key = (int(fm), int(fp), int(pid))
            if key not in sig_cache:
                sig_cache[key] = oracle_sigma(np.asarray(elem.face_barycentrics), *key[:2], PERMS[key[2]])
            sigma = sig_cache[key]
            vmap_plus[km, fm] = kp * n_p + fnodes[fp][sigma]
            vmap_plus[kp, fp] = km * n_p + fnodes[fm][np.argsort(sigma)]
        is_boundary = np.zeros((k_total, 4), dtype=bool)
        for k, f in self.boundary:
            is_boundary[k, f] = True
        self.vmap_minus, self.vmap_plus, self.is_boundary = vmap_minus, vmap_plus, is_boundary

    # oracle.py:50-58
    def face_states(self, u6: np.ndarray):
        flat = u6.reshape(6, -1)
        um = flat[:, self.vmap_minus]
        up = flat[:, self.vmap_plus]
        n = np.moveaxis(self.geo["normals"], -1, 0)[:, :, :, None]
        mirrored = pec_mirror(um, np.broadcast_to(n, (3,) + um.shape[1:]))
        up = np.where(self.is_boundary[None, :, :, None], mirrored, up)
        return um, up, n

    def volume(self, state: np.ndarray) -> np.ndarray:
        """(curl H / eps, -curl E / mu) alone (oracle.py:67-79, 91-93 without the lift)."""
        u = np.asarray(state, dtype=np.float64).reshape(6, self.num_elements, self.elem.num_nodes)
        ce, ch = self._curls(u)
        return np.concatenate([ch / self.eps, -ce / self.mu])

    def _curls(self, u):
        local = np.einsum("mij,fkj->mfki", self.elem.diff, u)
        grad = np.einsum("kmn,mfki->nfki", self.geo["drdx"], local)
        curl_e = np.stack([grad[1, 2] - grad[2, 1], grad[2, 0] - grad[0, 2], grad[0, 1] - grad[1, 0]])
        curl_h = np.stack([grad[1, 5] - grad[2, 4], grad[2, 3] - grad[0, 5], grad[0, 4] - grad[1, 3]])
        return curl_e, curl_h

    def scaled_flux(self, state: np.ndarray) -> np.ndarray:
        """upwind bracket * face Jacobian, (6, K, 4*Nfp) (oracle.py:82-85)."""
        u = np.asarray(state, dtype=np.float64).reshape(6, self.num_elements, self.elem.num_nodes)
        um, up, n = self.face_states(u)
        br = upwind_bracket(um, up, n, self.z, self.y)
        return (br * self.geo["sj"][None, :, :, None]).reshape(6, self.num_elements, -1)

    def rhs(self, state: np.ndarray) -> np.ndarray:
        """Semidiscrete RHS, natural (6, K, Np) (oracle.py:60-94)."""
        u = np.asarray(state, dtype=np.float64).reshape(6, self.num_elements, self.elem.num_nodes)
        curl_e, curl_h = self._curls(u)
        lifted = np.einsum("ij,fkj->fki", self.elem.lift, self.scaled_flux(u))
        lifted /= self.geo["det"][None, :, None]
        out = np.empty_like(u)
        out[0:3] = (curl_h + lifted[0:3]) / self.eps
        out[3:6] = (-curl_e + lifted[3:6]) / self.mu
        return out

    def energy(self, state: np.ndarray) -> float:
        """field_energy (maxwell.py:225-232)."""
        u = np.asarray(state)
        pf = np.einsum("fki,ij,fkj->fk", u, self.elem.mass, u) * self.geo["det"]
        return 0.5 * float(self.eps * pf[0:3].sum() + self.mu * pf[3:6].sum())


def build_oracle_operator(mesh, elem, eps: float = 1.0, mu: float = 1.0) -> OracleOperator:
    return OracleOperator(mesh.vertices, mesh.elements, elem, eps, mu)


def rk4_step(state, t: float, dt: float, rhs_fn):
    """Low-storage RK4 step (assemble.py:105-114)."""
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    y = np.array(state, dtype=np.float64, copy=True)
    r = np.zeros_like(y)
    for a, b, c in zip(RK_A, RK_B, RK_C):
        r = a * r + dt * np.asarray(rhs_fn(t + c * dt, y))
        y = y + b * r
    return y
