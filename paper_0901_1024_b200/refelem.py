"""Reference tetrahedron for the B200 operator: nodes, modal basis, local matrices.

Host-side setup, computed once per polynomial order and uploaded to HBM as the
kernels' constant operands.  The public names and conventions mirror the
reference package (``simtdg.refelem``) so existing callers work unchanged:

* bi-unit tet with vertices (-1,-1,-1), (1,-1,-1), (-1,1,-1), (-1,-1,1)
  (reference refelem.py:24-31), faces on t=-1, s=-1, r+s+t=-1, r=-1
  spanned by local vertices (0,1,2), (0,1,3), (1,2,3), (0,2,3) (refelem.py:34,356-358);
* true face areas [2, 2, 2*sqrt(3), 2] (refelem.py:49): the slanted face's mass
  matrix carries its own area factor;
* warp-and-blend interpolation nodes (Warburton 2006) in the reference's
  equidistant ordering (refelem.py:259-326);
* ``diff[mu] = (d_mu V) V^-1``, ``mass = V^-T V^-1``, ``lift = V V^T Embed``
  (refelem.py:371-446); ``face_nodes[f]`` sorted lexicographically on
  coordinates rounded to 10 digits (refelem.py:387-394);
* ``face_node_permutation`` pairs glued faces through barycentrics rounded to
  9 digits (refelem.py:449-467).

The implementation is independent: Jacobi polynomials come from the
normalised three-term recurrence instead of scipy's evaluator, the modal
gradients are written in the collapsed-coordinate chain rule directly, and the
face barycentrics are the closed-form affine coordinates of each face.  Every
array is pinned against the reference's own output (tests/golden/refelem.npz)
to 1e-12 and the integer tables bit for bit.
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np

REFERENCE_VERTICES = np.array(
    [[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]]
)
FACE_VERTEX_IDS = ((0, 1, 2), (0, 1, 3), (1, 2, 3), (0, 2, 3))
_INV_SQRT3 = 1.0 / math.sqrt(3.0)
FACE_UNIT_NORMALS = np.array(
    [[0.0, 0.0, -1.0], [0.0, -1.0, 0.0], [_INV_SQRT3, _INV_SQRT3, _INV_SQRT3], [-1.0, 0.0, 0.0]]
)
FACE_AREAS = np.array([2.0, 2.0, 2.0 * math.sqrt(3.0), 2.0])
NUM_FACES = 4
MAX_ORDER = 9

# Warburton's optimised blend exponents (one per order); orders <= 3 use none.
_BLEND_ALPHA = (0.0, 0.0, 0.0, 0.0, 0.1002, 1.1332, 1.5608, 1.3413, 1.2577, 1.1603)

_ON_FACE_TOL = 1e-8


def simplex_node_count(order: int) -> tuple[int, int]:
    """(Np, Nfp) of the degree-``order`` tetrahedron; ValueError for order < 1."""
    if order < 1:
        raise ValueError(f"polynomial order must be >= 1, got {order}")
    n = int(order)
    return (n + 1) * (n + 2) * (n + 3) // 6, (n + 1) * (n + 2) // 2


# ---------------------------------------------------------------------------
# Orthonormal Jacobi polynomials by recurrence


def _jacobi_table(x: np.ndarray, alpha: float, beta: float, nmax: int) -> np.ndarray:
    """Rows 0..nmax of the L2-orthonormal Jacobi polynomials P_n^(alpha,beta)(x)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty((nmax + 1,) + x.shape)
    ab = alpha + beta
    g0 = (2.0 ** (ab + 1.0) / (ab + 1.0) * math.gamma(alpha + 1.0)
          * math.gamma(beta + 1.0) / math.gamma(ab + 1.0))
    out[0] = 1.0 / math.sqrt(g0)
    if nmax == 0:
        return out
    g1 = (alpha + 1.0) * (beta + 1.0) / (ab + 3.0) * g0
    out[1] = ((ab + 2.0) * x / 2.0 + (alpha - beta) / 2.0) / math.sqrt(g1)
    a_prev = 2.0 / (2.0 + ab) * math.sqrt((alpha + 1.0) * (beta + 1.0) / (ab + 3.0))
    for i in range(1, nmax):
        h1 = 2.0 * i + ab
        a_next = 2.0 / (h1 + 2.0) * math.sqrt(
            (i + 1.0) * (i + 1.0 + ab) * (i + 1.0 + alpha) * (i + 1.0 + beta)
            / (h1 + 1.0) / (h1 + 3.0)
        )
        b_next = -(alpha * alpha - beta * beta) / h1 / (h1 + 2.0)
        out[i + 1] = ((x - b_next) * out[i] - a_prev * out[i - 1]) / a_next
        a_prev = a_next
    return out


def _jacobi(x, alpha: float, beta: float, n: int) -> np.ndarray:
    return _jacobi_table(x, alpha, beta, n)[n]


def _djacobi(x, alpha: float, beta: float, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros_like(np.asarray(x, dtype=np.float64))
    return math.sqrt(n * (n + alpha + beta + 1.0)) * _jacobi(x, alpha + 1.0, beta + 1.0, n - 1)


def _gauss_lobatto(p: int) -> np.ndarray:
    """Legendre-Gauss-Lobatto points on [-1, 1] (interior = roots of P^(1,1)_{p-1})."""
    if p == 1:
        return np.array([-1.0, 1.0])
    from scipy.special import roots_jacobi

    inner, _ = roots_jacobi(p - 1, 1.0, 1.0)
    return np.concatenate(([-1.0], np.sort(inner), [1.0]))


# ---------------------------------------------------------------------------
# Modal basis on the tetrahedron (collapsed coordinates a, b, c)


def _modes(order: int):
    return [(i, j, k) for i in range(order + 1)
            for j in range(order + 1 - i) for k in range(order + 1 - i - j)]


def _collapse(rst: np.ndarray):
    r, s, t = rst[:, 0], rst[:, 1], rst[:, 2]
    st = s + t
    safe_st = np.where(np.abs(st) > 1e-14, st, 1.0)
    a = np.where(np.abs(st) > 1e-14, -2.0 * (1.0 + r) / safe_st - 1.0, -1.0)
    omt = 1.0 - t
    safe_omt = np.where(np.abs(omt) > 1e-14, omt, 1.0)
    b = np.where(np.abs(omt) > 1e-14, 2.0 * (1.0 + s) / safe_omt - 1.0, -1.0)
    return a, b, t


def vandermonde(order: int, rst: np.ndarray) -> np.ndarray:
    """V[p, m] = phi_m(node_p) for the orthonormal Koornwinder-Dubiner basis."""
    a, b, c = _collapse(np.asarray(rst, dtype=np.float64))
    cols = []
    for i, j, k in _modes(order):
        cols.append(2.0 * math.sqrt(2.0) * _jacobi(a, 0.0, 0.0, i)
                    * _jacobi(b, 2.0 * i + 1.0, 0.0, j) * (1.0 - b) ** i
                    * _jacobi(c, 2.0 * (i + j) + 2.0, 0.0, k) * (1.0 - c) ** (i + j))
    return np.stack(cols, axis=1)


def grad_vandermonde(order: int, rst: np.ndarray) -> np.ndarray:
    """(3, n_nodes, n_modes): d/dr, d/ds, d/dt of every basis function."""
    a, b, c = _collapse(np.asarray(rst, dtype=np.float64))
    half_omb, half_omc = 0.5 * (1.0 - b), 0.5 * (1.0 - c)
    modes = _modes(order)
    out = np.empty((3, len(a), len(modes)))
    for m, (i, j, k) in enumerate(modes):
        pa, dpa = _jacobi(a, 0.0, 0.0, i), _djacobi(a, 0.0, 0.0, i)
        pb, dpb = _jacobi(b, 2.0 * i + 1.0, 0.0, j), _djacobi(b, 2.0 * i + 1.0, 0.0, j)
        ij = i + j
        pc = _jacobi(c, 2.0 * ij + 2.0, 0.0, k)
        dpc = _djacobi(c, 2.0 * ij + 2.0, 0.0, k)
        # d/da part (only through a), written with the (1-b)/2, (1-c)/2 weights
        fa = dpa * pb * pc
        if i > 0:
            fa = fa * half_omb ** (i - 1)
        if ij > 0:
            fa = fa * half_omc ** (ij - 1)
        # d/db part
        fb = dpb * half_omb ** i
        if i > 0:
            fb = fb - 0.5 * i * pb * half_omb ** (i - 1)
        if ij > 0:
            fb = fb * half_omc ** (ij - 1)
        fb = pa * fb * pc
        # d/dc part
        fc = dpc * half_omc ** ij
        if ij > 0:
            fc = fc - 0.5 * ij * pc * half_omc ** (ij - 1)
        fc = pa * pb * fc * half_omb ** i
        scale = 2.0 ** (2 * i + j + 1.5)
        dr = fa
        ds = 0.5 * (1.0 + a) * fa + fb
        dt = 0.5 * (1.0 + a) * fa + 0.5 * (1.0 + b) * fb + fc
        out[0, :, m] = dr * scale
        out[1, :, m] = ds * scale
        out[2, :, m] = dt * scale
    return out


def triangle_vandermonde(order: int, rs: np.ndarray) -> np.ndarray:
    """Orthonormal Dubiner basis on the bi-unit triangle, V[p, m]."""
    rs = np.asarray(rs, dtype=np.float64)
    r, s = rs[:, 0], rs[:, 1]
    oms = 1.0 - s
    a = np.where(np.abs(oms) > 1e-14, 2.0 * (1.0 + r) / np.where(np.abs(oms) > 1e-14, oms, 1.0) - 1.0, -1.0)
    cols = []
    for i in range(order + 1):
        for j in range(order + 1 - i):
            cols.append(math.sqrt(2.0) * _jacobi(a, 0.0, 0.0, i)
                        * _jacobi(s, 2.0 * i + 1.0, 0.0, j) * (1.0 - s) ** i)
    return np.stack(cols, axis=1)


# ---------------------------------------------------------------------------
# Warp-and-blend nodes


def _warp_1d(p: int, x: np.ndarray) -> np.ndarray:
    """Lagrange interpolant (equidistant -> GLL displacement), end roots deflated."""
    target = -_gauss_lobatto(p)
    xeq = 1.0 - 2.0 * np.arange(p + 1) / p
    w = np.zeros_like(x)
    for i in range(p + 1):
        term = np.full_like(x, target[i] - xeq[i])
        for j in range(1, p):
            if j != i:
                term = term * (x - xeq[j]) / (xeq[i] - xeq[j])
        if i != 0:
            term = -term / (xeq[i] - xeq[0])
        if i != p:
            term = term / (xeq[i] - xeq[p])
        w = w + term
    return w


def _face_warp(p: int, alpha: float, l1, l2, l3):
    """In-plane warp of one face in its equilateral frame (two components)."""
    w1 = l2 * l3 * 4.0 * _warp_1d(p, l3 - l2) * (1.0 + (alpha * l1) ** 2)
    w2 = l1 * l3 * 4.0 * _warp_1d(p, l1 - l3) * (1.0 + (alpha * l2) ** 2)
    w3 = l1 * l2 * 4.0 * _warp_1d(p, l2 - l1) * (1.0 + (alpha * l3) ** 2)
    c2, c4 = math.cos(2.0 * math.pi / 3.0), math.cos(4.0 * math.pi / 3.0)
    s2, s4 = math.sin(2.0 * math.pi / 3.0), math.sin(4.0 * math.pi / 3.0)
    return w1 + c2 * w2 + c4 * w3, s2 * w2 + s4 * w3


def warp_blend_nodes(order: int) -> np.ndarray:
    """(Np, 3) interpolation nodes on the reference tet, reference ordering."""
    n = int(order)
    alpha = _BLEND_ALPHA[n] if n < len(_BLEND_ALPHA) else 1.0
    # equidistant lattice: t-level outermost, then s, then r (refelem.py:259-266)
    lattice = np.array([(-1.0 + 2.0 * q / n, -1.0 + 2.0 * m / n, -1.0 + 2.0 * l / n)
                        for l in range(n + 1) for m in range(n + 1 - l)
                        for q in range(n + 1 - l - m)])
    r, s, t = lattice.T
    lam = {1: 0.5 * (1.0 + t), 2: 0.5 * (1.0 + s), 3: -0.5 * (1.0 + r + s + t), 4: 0.5 * (1.0 + r)}
    sq3, sq6 = math.sqrt(3.0), math.sqrt(6.0)
    v = {1: np.array([-1.0, -1.0 / sq3, -1.0 / sq6]), 2: np.array([1.0, -1.0 / sq3, -1.0 / sq6]),
         3: np.array([0.0, 2.0 / sq3, -1.0 / sq6]), 4: np.array([0.0, 0.0, 3.0 / sq6])}
    tangent1 = [v[2] - v[1], v[2] - v[1], v[3] - v[2], v[3] - v[1]]
    tangent2 = [v[3] - 0.5 * (v[1] + v[2]), v[4] - 0.5 * (v[1] + v[2]),
                v[4] - 0.5 * (v[2] + v[3]), v[4] - 0.5 * (v[1] + v[3])]
    tangent1 = [x / np.linalg.norm(x) for x in tangent1]
    tangent2 = [x / np.linalg.norm(x) for x in tangent2]
    xyz = (lam[3][:, None] * v[1] + lam[4][:, None] * v[2]
           + lam[2][:, None] * v[3] + lam[1][:, None] * v[4])
    shift = np.zeros_like(xyz)
    tol = 1e-10
    # (opposite-vertex coordinate, three in-face coordinates) per face
    faces = ((1, 2, 3, 4), (2, 1, 3, 4), (3, 1, 4, 2), (4, 1, 3, 2))
    for f, (ia, ib, ic, idd) in enumerate(faces):
        la, lb, lc, ld = lam[ia], lam[ib], lam[ic], lam[idd]
        wx, wy = _face_warp(n, alpha, lb, lc, ld)
        blend = lb * lc * ld
        denom = (lb + 0.5 * la) * (lc + 0.5 * la) * (ld + 0.5 * la)
        ok = denom > tol
        blend = np.where(ok, (1.0 + (alpha * la) ** 2) * blend / np.where(ok, denom, 1.0), blend)
        shift = shift + (blend * wx)[:, None] * tangent1[f] + (blend * wy)[:, None] * tangent2[f]
        inside = (lb > tol).astype(int) + (lc > tol) + (ld > tol)
        on_face = (la < tol) & (inside < 3)
        shift[on_face] = wx[on_face, None] * tangent1[f] + wy[on_face, None] * tangent2[f]
    xyz = xyz + shift
    # back to (r, s, t): xyz = v1*(l3) + ... is affine in rst
    amat = 0.5 * np.stack([v[2] - v[1], v[3] - v[1], v[4] - v[1]], axis=1)
    rhs = (xyz - 0.5 * (v[2] + v[3] + v[4] - v[1])).T
    return np.linalg.solve(amat, rhs).T


# ---------------------------------------------------------------------------
# Element assembly


@dataclass
class ReferenceElement:
    """Nodes and local operators of one order (arrays are read-only)."""

    order: int
    num_nodes: int
    num_face_nodes: int
    num_faces: int
    nodes: np.ndarray              # (Np, 3)
    vandermonde: np.ndarray        # (Np, Np)
    inv_vandermonde: np.ndarray    # (Np, Np)
    mass: np.ndarray               # (Np, Np)
    stiffness: np.ndarray          # (3, Np, Np)
    diff: np.ndarray               # (3, Np, Np)
    face_mass: np.ndarray          # (4, Nfp, Nfp), true surface measure
    lift: np.ndarray               # (Np, 4*Nfp)
    face_nodes: np.ndarray         # (4, Nfp) int64
    face_barycentrics: np.ndarray  # (4, Nfp, 3)


def _face_coordinates(f: int, nodes: np.ndarray):
    """Affine coordinates (u, w) of points on face f w.r.t. FACE_VERTEX_IDS corners."""
    r, s, t = nodes[:, 0], nodes[:, 1], nodes[:, 2]
    if f == 0:
        return 0.5 * (1.0 + r), 0.5 * (1.0 + s)
    if f == 1:
        return 0.5 * (1.0 + r), 0.5 * (1.0 + t)
    return 0.5 * (1.0 + s), 0.5 * (1.0 + t)  # faces 2 and 3 share the (s, t) chart


def _plane_distance(nodes: np.ndarray) -> np.ndarray:
    r, s, t = nodes[:, 0], nodes[:, 1], nodes[:, 2]
    return np.abs(np.stack([t + 1.0, s + 1.0, r + s + t + 1.0, r + 1.0]))


@functools.lru_cache(maxsize=None)
def build_reference_element(order: int) -> ReferenceElement:
    """All local matrices for ``order`` in 1..9 (ValueError otherwise).

    Cached per order: the instances are immutable.
    """
    if not 1 <= int(order) <= MAX_ORDER:
        raise ValueError(f"order must be in 1..{MAX_ORDER}, got {order}")
    order = int(order)
    n_p, n_fp = simplex_node_count(order)
    nodes = warp_blend_nodes(order)
    if nodes.shape != (n_p, 3):
        raise AssertionError("node construction produced a wrong count")
    vdm = vandermonde(order, nodes)
    cond = np.linalg.cond(vdm)
    if cond > 1e12:
        raise ValueError(f"Vandermonde matrix numerically singular (cond={cond:.3g})")
    vinv = np.linalg.inv(vdm)
    mass = vinv.T @ vinv
    gv = grad_vandermonde(order, nodes)
    diff = np.stack([gv[d] @ vinv for d in range(3)])
    stiff = np.stack([mass @ diff[d] for d in range(3)])

    dist = _plane_distance(nodes)
    face_nodes = np.empty((NUM_FACES, n_fp), dtype=np.int64)
    bary = np.empty((NUM_FACES, n_fp, 3))
    fmass = np.empty((NUM_FACES, n_fp, n_fp))
    for f in range(NUM_FACES):
        ids = np.flatnonzero(dist[f] < _ON_FACE_TOL)
        if ids.size != n_fp:
            raise AssertionError(f"face {f}: found {ids.size} nodes, expected {n_fp}")
        key = np.round(nodes[ids], 10)
        ids = ids[np.lexsort((key[:, 2], key[:, 1], key[:, 0]))]
        face_nodes[f] = ids
        u, w = _face_coordinates(f, nodes[ids])
        bary[f, :, 0] = 1.0 - u - w
        bary[f, :, 1] = u
        bary[f, :, 2] = w
        v2 = triangle_vandermonde(order, np.column_stack([2.0 * u - 1.0, 2.0 * w - 1.0]))
        fmass[f] = 0.5 * FACE_AREAS[f] * np.linalg.inv(v2 @ v2.T)

    embed = np.zeros((n_p, NUM_FACES * n_fp))
    for f in range(NUM_FACES):
        embed[face_nodes[f], f * n_fp:(f + 1) * n_fp] += fmass[f]
    lift = vdm @ (vdm.T @ embed)

    arrays = dict(nodes=nodes, vandermonde=vdm, inv_vandermonde=vinv, mass=mass,
                  stiffness=stiff, diff=diff, face_mass=fmass, lift=lift,
                  face_nodes=face_nodes, face_barycentrics=bary)
    for arr in arrays.values():
        arr.setflags(write=False)
    return ReferenceElement(order=order, num_nodes=n_p, num_face_nodes=n_fp,
                            num_faces=NUM_FACES, **arrays)


def build_lifting_matrix(elem: ReferenceElement) -> np.ndarray:
    """LIFT = V V^T Embed, Embed holding each face mass at its face-node rows."""
    n_p, n_fp = elem.num_nodes, elem.num_face_nodes
    embed = np.zeros((n_p, NUM_FACES * n_fp))
    for f in range(NUM_FACES):
        embed[elem.face_nodes[f], f * n_fp:(f + 1) * n_fp] += elem.face_mass[f]
    return elem.vandermonde @ (elem.vandermonde.T @ embed)


@functools.lru_cache(maxsize=None)
def _sigma_cached(order: int, face_minus: int, face_plus: int, vertex_perm: tuple) -> np.ndarray:
    elem = build_reference_element(order)
    bm = np.round(elem.face_barycentrics[face_minus], 9)
    bp = np.round(elem.face_barycentrics[face_plus][:, list(vertex_perm)], 9)
    index = {tuple(row): j for j, row in enumerate(bp)}
    try:
        sigma = np.array([index[tuple(row)] for row in bm], dtype=np.int64)
    except KeyError as exc:
        raise ValueError("face node sets do not match under the given vertex pairing") from exc
    sigma.setflags(write=False)
    return sigma


def face_node_permutation(elem: ReferenceElement, face_minus: int, face_plus: int,
                          vertex_perm) -> np.ndarray:
    """sigma with face_nodes[face_plus][sigma[i]] coincident with face_nodes[face_minus][i].

    ``vertex_perm[j]`` is the corner position on the plus face that matches
    corner ``j`` of the minus face (reference refelem.py:449-467).
    """
    if elem is build_reference_element(elem.order):
        return _sigma_cached(elem.order, int(face_minus), int(face_plus),
                             tuple(int(x) for x in vertex_perm)).copy()
    bm = np.round(elem.face_barycentrics[face_minus], 9)
    bp = np.round(elem.face_barycentrics[face_plus][:, list(vertex_perm)], 9)
    index = {tuple(row): j for j, row in enumerate(bp)}
    try:
        return np.array([index[tuple(row)] for row in bm], dtype=np.int64)
    except KeyError as exc:
        raise ValueError("face node sets do not match under the given vertex pairing") from exc
