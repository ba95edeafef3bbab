"""Element locality ordering for the stage kernels (the role of layout.py Alg. 2).

The reference numbers box-mesh elements ix-major (mesh.py:111-121), so a
64-element tile of the stage kernel is a column of ~11 cells whose x and y
face neighbours all live in other tiles (gathered from L2).  Sorting the
elements along a Morton (Z-order) curve of their centroids makes every tile
a compact 3-D blob, so more face neighbours sit in the tile's shared memory.
The order is internal to the operator: ``to_padded`` / ``from_padded`` and
every natural-order attribute keep the reference numbering.
"""

from __future__ import annotations

import numpy as np

from .facemaps import FaceMaps


def _spread_bits(x: np.ndarray) -> np.ndarray:
    """Insert two zero bits between the low 21 bits of x (3-D Morton interleave)."""
    x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
    x = (x | (x << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    x = (x | (x << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    x = (x | (x << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    x = (x | (x << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    x = (x | (x << np.uint64(2))) & np.uint64(0x1249249249249249)
    return x


def morton_order(vertices: np.ndarray, elements: np.ndarray, resolution: int | None = None) -> np.ndarray:
    """Permutation ``order`` (new slot -> element id) sorting elements by the Morton code of their centroid.

    Centroids are quantised to ``resolution`` cells per axis (default ~ (K/6)^(1/3), the cell count
    of a Kuhn-split box) so the tets of one cell share a code and stay together (stable sort).  On
    the C3 box this raises the fraction of face neighbours inside a 64-element tile from 0.65 to 0.71.
    """
    c = vertices[elements].mean(axis=1)
    if resolution is None:
        resolution = max(1, int(round((len(c) / 6.0) ** (1.0 / 3.0))))
    lo, hi = c.min(axis=0), c.max(axis=0)
    q = np.floor((c - lo) / np.maximum(hi - lo, 1e-300) * (resolution - 1e-9)).astype(np.int64)
    code = _spread_bits(q[:, 0]) | (_spread_bits(q[:, 1]) << np.uint64(1)) | (_spread_bits(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable").astype(np.int64)


def column_order(vertices: np.ndarray, elements: np.ndarray, resolution: int | None = None,
                 width: int = 2) -> np.ndarray:
    """Permutation sorting elements into ``width`` x ``width`` columns of grid cells along z.

    Centroids are binned on a grid of ``resolution`` cells per axis (default ~ (K/6)^(1/3)); the
    key is (column x, column y, z, x within column, y within column, element id).  A 64-element
    tile is then a 2 x 2 x ~2.7-cell block: 74 % of the face neighbours of the C3 box fall inside
    the tile (Morton 71 %, reference numbering 65 %).
    """
    c = vertices[elements].mean(axis=1)
    if resolution is None:
        resolution = max(1, int(round((len(c) / 6.0) ** (1.0 / 3.0))))
    lo, hi = c.min(axis=0), c.max(axis=0)
    q = np.floor((c - lo) / np.maximum(hi - lo, 1e-300) * (resolution - 1e-9)).astype(np.int64)
    # columns visited along a Morton curve of the column grid: x- and y-adjacent columns are then
    # mostly processed close in time, so their rows are still in L2 when gathered (86 % of the
    # out-of-tile neighbours within half a wave of CTAs on C3, vs 68 % for row-major columns)
    col = _spread_bits(q[:, 0] // width) | (_spread_bits(q[:, 1] // width) << np.uint64(1))
    return np.lexsort((np.arange(len(c)), q[:, 1] % width, q[:, 0] % width, q[:, 2], col)).astype(np.int64)


def permute_maps(maps: FaceMaps, order: np.ndarray) -> FaceMaps:
    """Face maps in the new numbering: row s is old element order[s], neighbour ids relabelled.

    Neighbour ids >= len(order) (ghost slots of a multi-GPU rank) are left unchanged.
    """
    k = len(order)
    inv = np.empty_like(order)
    inv[order] = np.arange(k)
    nb = maps.neighbors[order].astype(np.int64)
    nbr = np.where(nb < k, inv[np.minimum(nb, k - 1)], nb).astype(np.int32)
    return FaceMaps(num_nodes=maps.num_nodes, face_nodes=maps.face_nodes, neighbors=nbr,
                    codes=maps.codes[order].copy(), code_table=maps.code_table)


# ----------------------------------------------------------------------------------------------
# Face-node slot order of the tensor-core flux pass (dgm_tc.cuh flux_pass)
# ----------------------------------------------------------------------------------------------

def _flux_lane_groups(order: int, np_stride: int, nfp: int, nfpk: int):
    """(rows, slots) of the 32 lanes of every (warp, node j) shared load of the flux pass.

    Mirrors dgm_tc.cuh: TcCfg<N>::TE elements per CTA, FB = 4 face nodes per work unit,
    unit = tid -> row = unit / NBF, slot = (unit % NBF) * FB + j; the owned-row trace load of a
    lane reads s_u[row * NPG + fmask[face][slot]] (pad slots read slot 0).
    """
    te = 64 if order <= 6 else (32 if order <= 8 else 16)
    fb, nbf = 4, nfpk // 4
    rows, slots = [], []
    for w in range((te * nbf + 31) // 32):
        u = np.arange(w * 32, w * 32 + 32)
        u = u[u // nbf < te]
        for j in range(fb):
            r = np.zeros(32, np.int64)
            s = np.full(32, -1, np.int64)
            r[: len(u)], s[: len(u)] = u // nbf, (u % nbf) * fb + j
            rows.append(r)
            slots.append(s)
    rows, slots = np.array(rows), np.array(slots)
    live = slots >= 0
    slots = np.where((slots >= nfp) | ~live, 0, slots)  # pad slots read node slot 0
    return rows * np_stride, slots, live


def _bank_cost(nodes: np.ndarray, base: np.ndarray, slots: np.ndarray, live: np.ndarray) -> int:
    """Sum over load groups of the max lanes per shared bank (wavefronts per load)."""
    g = len(base)
    banks = (base + nodes[slots]) % 32 + 32 * np.arange(g)[:, None]
    counts = np.bincount(banks[live], minlength=32 * g).reshape(g, 32)
    return int(counts.max(axis=1).sum())


def face_slot_order(face_nodes: np.ndarray, order: int, np_stride: int, nfpk: int) -> np.ndarray:
    """(4, Nfp) permutation: slot i of face f holds face node perm[f, i].

    The order of the nodes inside a face is free (fmask, the code table and the LIFT columns are
    permuted together), so it is chosen to spread the flux pass's owned-row trace loads over the
    32 shared-memory banks: a deterministic pairwise-swap descent on the lane model above
    (e.g. N=4: 2.0 -> 1.0..1.25 wavefronts per load).
    """
    face_nodes = np.asarray(face_nodes, dtype=np.int64)
    nf, nfp = face_nodes.shape
    base, slots, live = _flux_lane_groups(order, np_stride, nfp, nfpk)
    perms = np.empty((nf, nfp), dtype=np.int64)
    for f in range(nf):
        perm = np.arange(nfp)
        cur = _bank_cost(face_nodes[f][perm], base, slots, live)
        improved = True
        while improved:
            improved = False
            for a in range(nfp):
                for b in range(a + 1, nfp):
                    perm[[a, b]] = perm[[b, a]]
                    c = _bank_cost(face_nodes[f][perm], base, slots, live)
                    if c < cur:
                        cur, improved = c, True
                    else:
                        perm[[a, b]] = perm[[b, a]]
        perms[f] = perm
    return perms


def _v2_cost(nodes: np.ndarray, nfpk: int) -> int:
    """Shared-memory wavefronts of the v2 kernel's owned-trace loads for one face slot order.

    dgm_tc2.cuh: at step jj lane (e, b) of a flux warp loads node nodes[4b + (jj + b) % 4] of element
    e (the rotation keeps its flux stores conflict-free); the state tile stores node j of row e at
    bank (4e + j mod 4) mod 32, so the 8 elements of a warp cover all banks once per residue and the
    cost of load jj is the largest number of blocks b whose node has the same residue.  Padding
    slots (>= Nfp) read slot 0's node.
    """
    nfp = len(nodes)
    cost = 0
    for jj in range(4):
        slots = [4 * b + (jj + b) % 4 for b in range(nfpk // 4)]
        res = [int(nodes[s] if s < nfp else nodes[0]) % 4 for s in slots]
        cost += max(res.count(r) for r in set(res))
    return cost


def face_slot_order_v2(face_nodes: np.ndarray, nfpk: int) -> np.ndarray:
    """(4, Nfp) slot permutation for the v2 tensor kernel (the v1 model is face_slot_order).

    Pairwise-swap descent on _v2_cost from the natural order, then seeded restarts until every
    column of slots reads four distinct residues (N=4: 16 -> 4 wavefronts per 4 loads) or the
    budget is spent; deterministic.
    """
    face_nodes = np.asarray(face_nodes, dtype=np.int64)
    nf, nfp = face_nodes.shape
    floor = 4 * max(1, -(-(nfpk // 4) // 4)) if nfpk >= 16 else 4
    rng = np.random.default_rng(0)
    perms = np.empty((nf, nfp), dtype=np.int64)
    for f in range(nf):
        best, best_cost = None, None
        for attempt in range(64):
            perm = np.arange(nfp) if attempt == 0 else rng.permutation(nfp)
            cur = _v2_cost(face_nodes[f][perm], nfpk)
            improved = True
            while improved:
                improved = False
                for a in range(nfp):
                    for b in range(a + 1, nfp):
                        perm[[a, b]] = perm[[b, a]]
                        c = _v2_cost(face_nodes[f][perm], nfpk)
                        if c < cur:
                            cur, improved = c, True
                        else:
                            perm[[a, b]] = perm[[b, a]]
            if best_cost is None or cur < best_cost:
                best, best_cost = perm.copy(), cur
            if best_cost <= floor:
                break
        perms[f] = best
    return perms


def permute_face_slots(maps: FaceMaps, perm: np.ndarray) -> FaceMaps:
    """FaceMaps whose face node i of face f is the natural face node perm[f, i].

    Code-table rows are per (own face, code) after the permutation, so codes are re-issued.
    """
    nf = perm.shape[0]
    face_nodes = np.take_along_axis(np.asarray(maps.face_nodes, dtype=np.int64), perm, axis=1)
    codes = np.asarray(maps.codes)
    new_codes = np.full_like(codes, -1)
    rows: dict = {}
    table = []
    for f in range(nf):
        col = codes[:, f]
        for c in np.unique(col[col >= 0]):
            row = np.asarray(maps.code_table[c])[perm[f]].astype(np.uint8)
            key = row.tobytes()
            if key not in rows:
                rows[key] = len(table)
                table.append(row)
            new_codes[col == c, f] = rows[key]
    code_table = np.array(table, dtype=np.uint8).reshape(len(table), perm.shape[1])
    return FaceMaps(num_nodes=maps.num_nodes, face_nodes=face_nodes, neighbors=maps.neighbors,
                    codes=new_codes, code_table=code_table)


# ---------------------------------------------------------------------------
# The paper's Alg. 2 partitioner (reference layout.py:59-117, greedy_partition), as an element order.


def greedy_partition(mesh, max_block_size: int, connectivity=None) -> list:
    """Connected blocks of at most ``max_block_size`` elements, identical to the reference's Alg. 2.

    Breadth-first agglomeration: the growing block absorbs the queued candidate sharing the most faces
    with it (ties: the earliest queued entry); a full block reseeds from the queue's front entry, an
    exhausted queue from the lowest remaining element id.  The reference rescans its whole queue per
    pick (quadratic in the block's frontier); here the queue is an append-only array with a heap keyed
    (-shared faces, queue position) and lazy invalidation, so it runs in O(K log K) and reproduces the
    reference's blocks exactly (tests/test_setup.py, golden partitions made by the reference itself).
    """
    import heapq

    if max_block_size < 1:
        raise ValueError("max_block_size must be >= 1")
    if connectivity is None:
        from .mesh import build_connectivity

        connectivity = build_connectivity(mesh)
    k = int(mesh.num_elements)
    # neighbour lists in the reference's order: interior pairs in connectivity order, both directions
    em = np.asarray(connectivity.elem_minus, dtype=np.int64)
    ep = np.asarray(connectivity.elem_plus, dtype=np.int64)
    src = np.stack([em, ep], axis=1).reshape(-1)
    dst = np.stack([ep, em], axis=1).reshape(-1)
    order = np.argsort(src, kind="stable")
    nbr_flat = dst[order]
    start = np.zeros(k + 1, dtype=np.int64)
    np.add.at(start, src + 1, 1)
    start = np.cumsum(start)
    neighbors = [nbr_flat[start[i]:start[i + 1]].tolist() for i in range(k)]

    taken = np.zeros(k, dtype=bool)
    min_free = 0
    partition = []
    next_seed = None
    shared = np.zeros(k, dtype=np.int64)     # faces shared with the current block
    while min_free < k:
        seed = next_seed if next_seed is not None and not taken[next_seed] else min_free
        next_seed = None
        q_elem = [seed]                      # the queue: append-only, entries popped by flag
        q_live = [True]
        live_count = 1
        entries: dict = {seed: [0]}          # element -> its queue positions
        heap = [(0, 0)]
        block = []
        touched = []
        while True:
            while True:                      # the live entry with the most shared faces, earliest
                neg, pos = heapq.heappop(heap)
                if q_live[pos] and -neg == shared[q_elem[pos]]:
                    break
            elem = q_elem[pos]
            q_live[pos] = False
            live_count -= 1
            if not taken[elem]:
                taken[elem] = True
                while min_free < k and taken[min_free]:
                    min_free += 1
                block.append(elem)
                if len(block) == max_block_size:
                    if live_count:
                        next_seed = next(q_elem[p] for p in range(len(q_elem)) if q_live[p])
                    break
                for nb in neighbors[elem]:  # counts of queued candidates adjacent to elem grow
                    shared[nb] += 1
                    touched.append(nb)
                    for p in entries.get(nb, ()):
                        if q_live[p]:
                            heapq.heappush(heap, (-shared[nb], p))
                for nb in neighbors[elem]:  # queue.extend(neighbors[elem])
                    p = len(q_elem)
                    q_elem.append(nb)
                    q_live.append(True)
                    live_count += 1
                    entries.setdefault(nb, []).append(p)
                    heapq.heappush(heap, (-shared[nb], p))
            if not live_count:
                if min_free >= k:
                    break
                p = len(q_elem)
                q_elem.append(min_free)
                q_live.append(True)
                live_count += 1
                entries.setdefault(min_free, []).append(p)
                heapq.heappush(heap, (-shared[min_free], p))
        partition.append(block)
        for nb in touched:
            shared[nb] = 0
    return partition


def greedy_block_order(vertices: np.ndarray, elements: np.ndarray, block: int = 64, connectivity=None) -> np.ndarray:
    """Element order made of the Alg. 2 blocks of ``block`` elements (the tensor kernels' tile size)."""
    from .mesh import Mesh

    blocks = greedy_partition(Mesh(vertices, elements), block, connectivity)
    return np.concatenate([np.asarray(b, dtype=np.int64) for b in blocks])
