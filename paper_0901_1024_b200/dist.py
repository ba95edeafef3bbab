"""Element-partitioned multi-GPU operator: one rank per B200, face-trace halo over NVLink.

The reference is single-process; this module adds the one
parallel strategy the operator admits: contiguous element
ranges per rank.  Box meshes are numbered ix-major (reference mesh.py:111-121),
so a contiguous range of whole x-layers of cells is an x-slab and its only
neighbours are the two adjacent slabs.

Per rank (``RankDomain``):
  * owned elements get local ids 0..K_own-1 (global order preserved), ghosts
    (neighbours owned elsewhere) get K_own.. sorted by global id, i.e. grouped
    by owning rank;
  * ``send[peer]``: local ids of owned elements that are ghosts on ``peer``,
    in the order the peer stores them; ``recv[peer] = (ghost_begin, count)``;
  * ``interior = (p, q)``: a contiguous owned range none of whose elements
    reads a ghost -- the stage kernel runs on it while the halo is in flight.

Per LSRK stage (``DistributedMaxwellOperator``): on a communication stream,
pack the boundary elements of u_in (dgm_halo_pack), exchange with NCCL
send/recv, unpack into the ghost slots (dgm_halo_unpack); meanwhile the
compute stream runs the fused stage kernel on the interior range; then the
boundary ranges.  Only scalar diagnostics use an all-reduce.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .facemaps import FaceMaps, build_face_maps
from .maxwell import VACUUM, Material
from .mesh import Mesh, box_slab_mesh, build_connectivity, compute_geometry, map_nodes
from .refelem import NUM_FACES, ReferenceElement


def split_range(n: int, parts: int, index: int) -> tuple[int, int]:
    """Balanced contiguous split of range(n) into ``parts``; returns part ``index``."""
    base, extra = divmod(int(n), int(parts))
    begin = index * base + min(index, extra)
    return begin, begin + base + (1 if index < extra else 0)


@dataclass
class RankDomain:
    rank: int
    world: int
    elem: ReferenceElement
    owned: tuple[int, int]          # global element range [g0, g1)
    ghost_global: np.ndarray        # (G,) global ids of ghosts, sorted
    maps: FaceMaps                  # neighbors in local ids (owned + ghost range)
    geo_words: np.ndarray           # (K_own, 26)
    det_j: np.ndarray               # (K_own,)
    send: dict = field(default_factory=dict)   # peer -> local owned ids (int32)
    recv: dict = field(default_factory=dict)   # peer -> (ghost_begin, count)
    interior: tuple[int, int] = (0, 0)
    # face-trace halo: peer -> int32 (n, 2) (local element, face) pairs, the same cut faces in the
    # same order on both ends (sorted by the face owner's global id, then face)
    send_traces: dict = field(default_factory=dict)   # owned element's face whose neighbour is on peer
    recv_traces: dict = field(default_factory=dict)   # ghost slot's face whose neighbour is owned here
    owner_ranges: list = field(default_factory=list)  # per rank global [g0, g1)
    mesh: Mesh | None = None        # submesh holding owned (+ ghost) elements
    sub_offset: int = 0             # submesh element j <-> global j + sub_offset

    @property
    def num_owned(self) -> int:
        return self.owned[1] - self.owned[0]

    @property
    def num_ghost(self) -> int:
        return len(self.ghost_global)

    def owned_nodes(self) -> np.ndarray:
        """(K_own, Np, 3) physical node coordinates of the owned elements."""
        lo = self.owned[0] - self.sub_offset
        sub = Mesh(self.mesh.vertices, self.mesh.elements[lo:lo + self.num_owned])
        return map_nodes(sub, self.elem)


def _localize(rank: int, world: int, owner_ranges, nbr_global: np.ndarray, codes: np.ndarray,
              owned: tuple[int, int]):
    """Map owned rows' global neighbor ids to local ids; derive ghosts, recv slices, interior range."""
    g0, g1 = owned
    k_own = g1 - g0
    inner = codes >= 0
    outside = inner & ((nbr_global < g0) | (nbr_global >= g1))
    ghost_global = np.unique(nbr_global[outside])
    local = nbr_global.astype(np.int64) - g0
    if len(ghost_global):
        local[outside] = k_own + np.searchsorted(ghost_global, nbr_global[outside])
    local[~inner] = np.arange(k_own)[:, None].repeat(NUM_FACES, 1)[~inner]
    recv = {}
    for peer, (p0, p1) in enumerate(owner_ranges):
        if peer == rank:
            continue
        lo, hi = np.searchsorted(ghost_global, [p0, p1])
        if hi > lo:
            recv[peer] = (k_own + int(lo), int(hi - lo))
    touches = outside.any(axis=1)
    idx = np.flatnonzero(touches)
    if len(idx) == 0:
        interior = (0, k_own)
    else:
        # largest gap between boundary elements is the interior range
        edges = np.concatenate(([-1], idx, [k_own]))
        gaps = np.diff(edges) - 1
        j = int(np.argmax(gaps))
        interior = (int(edges[j] + 1), int(edges[j + 1]))
    return local.astype(np.int32), ghost_global.astype(np.int64), recv, interior


def _send_lists(rank: int, world: int, owned, owner_ranges, ghost_lists_of_peers):
    """Local ids this rank must send to each peer (peer's ghosts owned here, sorted)."""
    g0, g1 = owned
    send = {}
    for peer, ghosts in ghost_lists_of_peers.items():
        if peer == rank:
            continue
        mine = ghosts[(ghosts >= g0) & (ghosts < g1)]
        if len(mine):
            send[peer] = (mine - g0).astype(np.int32)
    return send


def _cut_traces(elem_ids: np.ndarray, nbr_g: np.ndarray, codes: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """(global element id, face) of the listed element rows whose face neighbour lies in [lo, hi).

    Rows come in ascending global id and np.nonzero walks them row-major, so the pairs are sorted
    by (element, face): sender and receiver enumerate the same cut faces in the same order.
    """
    e, f = np.nonzero((codes >= 0) & (nbr_g >= lo) & (nbr_g < hi))
    return np.stack([np.asarray(elem_ids, dtype=np.int64)[e], f.astype(np.int64)], axis=1)


def _trace_lists(rank: int, owned, owner_ranges, ghost_global, peers, rows_of):
    """send_traces / recv_traces of a rank; rows_of(global ids) -> (nbr_global, codes) of those elements."""
    g0, g1 = owned
    k_own = g1 - g0
    own_ids = np.arange(g0, g1)
    own_nbr, own_codes = rows_of(own_ids)
    send, recv = {}, {}
    for peer in peers:
        p0, p1 = owner_ranges[peer]
        out = _cut_traces(own_ids, own_nbr, own_codes, p0, p1)
        if len(out):
            out[:, 0] -= g0
            send[peer] = out.astype(np.int32)
        gh = ghost_global[(ghost_global >= p0) & (ghost_global < p1)]
        if len(gh):
            nbr, codes = rows_of(gh)
            inn = _cut_traces(gh, nbr, codes, g0, g1)
            inn[:, 0] = k_own + np.searchsorted(ghost_global, inn[:, 0])
            recv[peer] = inn.astype(np.int32)
    return send, recv


def _geometry_rows(mesh: Mesh, rows: slice):
    from .operator import geometry_words

    sub = Mesh(mesh.vertices, mesh.elements[rows])
    geo = compute_geometry(sub)
    return geometry_words(geo), geo.det_jacobians


def build_box_domain(extent, cells, elem: ReferenceElement, rank: int, world: int) -> RankDomain:
    """Rank ``rank`` of an x-slab partition of generate_box_mesh(extent, cells), set up locally.

    Each rank meshes only its slab plus one ghost cell layer on each side
    (O(K/P) host work), which reproduces the global connectivity exactly for
    the owned elements (tests/test_dist.py).
    """
    nx, ny, nz = (int(c) for c in cells)
    if world > nx:
        raise ValueError(f"{world} ranks need at least {world} cell layers in x, got {nx}")
    per_layer = ny * nz * 6
    layer_ranges = [split_range(nx, world, r) for r in range(world)]
    owner_ranges = [(a * per_layer, b * per_layer) for a, b in layer_ranges]
    ix0, ix1 = layer_ranges[rank]
    lo, hi = max(ix0 - 1, 0), min(ix1 + 1, nx)
    sub = box_slab_mesh(extent, cells, lo, hi)
    off = lo * per_layer
    conn = build_connectivity(sub)
    maps_sub = build_face_maps(sub, elem, conn)
    own = slice((ix0 - lo) * per_layer, (ix1 - lo) * per_layer)
    owned = owner_ranges[rank]
    nbr_g = maps_sub.neighbors[own].astype(np.int64) + off
    codes = maps_sub.codes[own].copy()
    # faces on the slab mesh's artificial x-walls belong to ghost elements only
    local, ghosts, recv, interior = _localize(rank, world, owner_ranges, nbr_g, codes, owned)
    # a peer's ghosts owned here: my elements with a face neighbor in the peer's range
    # (face adjacency is symmetric), in global order -- the order the peer stores them
    send = {}
    for peer in (rank - 1, rank + 1):
        if 0 <= peer < world:
            p0, p1 = owner_ranges[peer]
            touching = ((nbr_g >= p0) & (nbr_g < p1) & (codes >= 0)).any(axis=1)
            rows = np.flatnonzero(touching)
            if len(rows):
                send[peer] = rows.astype(np.int32)
    geo_words, det = _geometry_rows(sub, own)
    maps = FaceMaps(num_nodes=elem.num_nodes, face_nodes=maps_sub.face_nodes, neighbors=local, codes=codes,
                    code_table=maps_sub.code_table)

    def rows_of(ids):  # the slab mesh holds the owned and the ghost-layer elements' full face data
        j = np.asarray(ids, dtype=np.int64) - off
        return maps_sub.neighbors[j].astype(np.int64) + off, maps_sub.codes[j]

    peers = [p for p in (rank - 1, rank + 1) if 0 <= p < world]
    send_tr, recv_tr = _trace_lists(rank, owned, owner_ranges, ghosts, peers, rows_of)
    return RankDomain(rank=rank, world=world, elem=elem, owned=owned, ghost_global=ghosts, maps=maps,
                      geo_words=geo_words, det_j=det, send=send, recv=recv, interior=interior,
                      send_traces=send_tr, recv_traces=recv_tr,
                      owner_ranges=owner_ranges, mesh=sub, sub_offset=off)


def build_mesh_domain(mesh: Mesh, elem: ReferenceElement, rank: int, world: int,
                      global_maps: FaceMaps | None = None) -> RankDomain:
    """Generic partition: contiguous element ranges of an arbitrary mesh (global setup on every rank)."""
    k = mesh.num_elements
    owner_ranges = [split_range(k, world, r) for r in range(world)]
    maps_g = build_face_maps(mesh, elem) if global_maps is None else global_maps
    owned = owner_ranges[rank]
    rows = slice(*owned)
    nbr_g = maps_g.neighbors[rows].astype(np.int64)
    codes = maps_g.codes[rows].copy()
    local, ghosts, recv, interior = _localize(rank, world, owner_ranges, nbr_g, codes, owned)
    ghost_lists = {}
    for peer in range(world):
        if peer == rank:
            continue
        p0, p1 = owner_ranges[peer]
        pn, pc = maps_g.neighbors[p0:p1].astype(np.int64), maps_g.codes[p0:p1]
        out = (pc >= 0) & ((pn < p0) | (pn >= p1))
        ghost_lists[peer] = np.unique(pn[out])
    send = _send_lists(rank, world, owned, owner_ranges, ghost_lists)
    geo_words, det = _geometry_rows(mesh, rows)
    maps = FaceMaps(num_nodes=elem.num_nodes, face_nodes=maps_g.face_nodes, neighbors=local, codes=codes,
                    code_table=maps_g.code_table)

    def rows_of(ids):
        j = np.asarray(ids, dtype=np.int64)
        return maps_g.neighbors[j].astype(np.int64), maps_g.codes[j]

    send_tr, recv_tr = _trace_lists(rank, owned, owner_ranges, ghosts, [p for p in range(world) if p != rank],
                                    rows_of)
    return RankDomain(rank=rank, world=world, elem=elem, owned=owned, ghost_global=ghosts, maps=maps,
                      geo_words=geo_words, det_j=det, send=send, recv=recv, interior=interior,
                      send_traces=send_tr, recv_traces=recv_tr,
                      owner_ranges=owner_ranges, mesh=mesh, sub_offset=0)


class DistributedMaxwellOperator:
    """One rank's share of the operator; halo exchange over torch.distributed (NCCL)."""

    def __init__(self, domain: RankDomain, material: Material = VACUUM, *, dtype=None, device=None,
                 path: str = "auto", reorder: bool | None = None, face_slots: bool | None = None):
        import torch

        from .operator import B200MaxwellOperator

        self.domain = domain
        self.torch = torch
        dtype = torch.float32 if dtype is None else dtype
        if reorder is None:
            reorder = 2 <= domain.elem.order <= 8  # as build_b200_operator
        self.op = B200MaxwellOperator(domain.elem, material, domain.geo_words, domain.det_j, domain.maps,
                                      num_ghost=domain.num_ghost, dtype=dtype, device=device, path=path,
                                      order=self._interior_order(domain) if reorder else None,
                                      face_slots=face_slots)
        self.device = self.op.device
        self.comm_stream = torch.cuda.Stream(self.device)
        # face-trace halo buffers: 6 x Nfp reals per cut face (not whole ghost rows)
        width = 6 * domain.elem.num_face_nodes
        self._send = {p: (torch.as_tensor(np.ascontiguousarray(tr), device=self.device),
                          torch.empty((len(tr), width), dtype=dtype, device=self.device))
                      for p, tr in domain.send_traces.items()}
        self._recv_lists = {p: torch.as_tensor(np.ascontiguousarray(tr), device=self.device)
                            for p, tr in domain.recv_traces.items()}
        self._recv = {p: torch.empty((len(tr), width), dtype=dtype, device=self.device)
                      for p, tr in domain.recv_traces.items()}
        self._alt = self.op.empty_state()
        self._alt2 = self.op.empty_state()
        self._res = self.op.empty_state()

    @staticmethod
    def _interior_order(domain: RankDomain) -> np.ndarray:
        """Locality order (ordering.column_order) of the interior range only.

        The boundary ranges, whose rows are sent to peers and which are launched after the halo
        arrives, keep their slots, so send lists, ghost slots and the interior / boundary split
        are unchanged.
        """
        from .ordering import column_order

        k = domain.num_owned
        p, q = domain.interior
        order = np.arange(k, dtype=np.int64)
        if q - p > 1:
            lo = domain.owned[0] - domain.sub_offset
            elems = domain.mesh.elements[lo + p:lo + q]
            order[p:q] = p + column_order(domain.mesh.vertices, elems)
        return order

    @property
    def num_elements(self) -> int:
        return self.op.num_elements

    def to_padded(self, natural_owned):
        """Owned natural (6, K_own, Np) -> padded local state (ghost slots zero until exchanged)."""
        return self.op.to_padded(natural_owned)

    def exchange(self, u) -> None:
        """Fill u's ghost slots from their owners (blocking on the current stream)."""
        ev = self._exchange_async(u)
        self.torch.cuda.current_stream(self.device).wait_event(ev)

    def pack(self, u, stream=None) -> dict:
        """dgm_trace_pack the cut-face traces of u for every peer; returns {peer: buffer}."""
        from . import _capi

        s = self.torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream.cuda_stream
        for peer, (pairs, buf) in self._send.items():
            _capi.check(self.op._lib.dgm_trace_pack(self.op._plan, u.data_ptr(), pairs.data_ptr(), len(pairs),
                                                    buf.data_ptr(), s), "dgm_trace_pack")
        return {peer: buf for peer, (_, buf) in self._send.items()}

    def unpack(self, u, stream=None) -> None:
        """dgm_trace_unpack every received trace buffer into the face nodes of u's ghost rows."""
        from . import _capi

        s = self.torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream.cuda_stream
        for peer, buf in self._recv.items():
            pairs = self._recv_lists[peer]
            _capi.check(self.op._lib.dgm_trace_unpack(self.op._plan, buf.data_ptr(), pairs.data_ptr(), len(pairs),
                                                      u.data_ptr(), s), "dgm_trace_unpack")

    @property
    def recv_buffers(self) -> dict:
        return self._recv

    def _exchange_async(self, u):
        """Pack -> NCCL send/recv -> unpack on the communication stream; returns its completion event."""
        torch = self.torch
        import torch.distributed as dist

        compute = torch.cuda.current_stream(self.device)
        self.comm_stream.wait_stream(compute)
        with torch.cuda.stream(self.comm_stream):
            sends = self.pack(u, self.comm_stream)
            if dist.is_initialized() and dist.get_backend() == "gloo":
                # gloo moves host tensors only: stage the (small) trace buffers through the host.  For
                # tests of the multi-rank paths on one GPU (NCCL refuses two ranks on one device).
                self.comm_stream.synchronize()
                host_recv = {p: torch.empty(b.shape, dtype=b.dtype) for p, b in self._recv.items()}
                ops = [dist.P2POp(dist.isend, buf.cpu(), peer) for peer, buf in sends.items()]
                ops += [dist.P2POp(dist.irecv, buf, peer) for peer, buf in host_recv.items()]
                if ops:
                    for req in dist.batch_isend_irecv(ops):
                        req.wait()
                for peer, buf in host_recv.items():
                    self._recv[peer].copy_(buf)
            else:
                ops = [dist.P2POp(dist.isend, buf, peer) for peer, buf in sends.items()]
                ops += [dist.P2POp(dist.irecv, buf, peer) for peer, buf in self._recv.items()]
                if ops:
                    for req in dist.batch_isend_irecv(ops):
                        req.wait()
            self.unpack(u, self.comm_stream)
            ev = torch.cuda.Event()
            ev.record(self.comm_stream)
        return ev

    def stage_ranges(self):
        """(interior range, boundary ranges) of the owned elements."""
        p, q = self.domain.interior
        k = self.op.num_elements
        bnd = [(a, b) for a, b in ((0, p), (q, k)) if b > a]
        return (p, q), bnd

    def _stage(self, u_in, u_out, a, b, dt) -> None:
        (p, q), boundary = self.stage_ranges()
        ev = self._exchange_async(u_in)
        if q > p:  # interior elements read no ghost: overlap with the halo exchange
            self.op.lsrk_stage(u_in, u_out, self._res, a, b, dt, p, q)
        self.torch.cuda.current_stream(self.device).wait_event(ev)
        for lo, hi in boundary:
            self.op.lsrk_stage(u_in, u_out, self._res, a, b, dt, lo, hi)

    def advance(self, u, dt: float, nsteps: int = 1):
        """nsteps LSRK4 steps of the owned elements (ghosts refreshed every stage)."""
        from .stepper import RK_A, RK_B

        if dt <= 0.0:
            raise ValueError("dt must be positive")
        for _ in range(int(nsteps)):  # u -> alt -> alt2 -> alt -> alt2 -> u, as B200MaxwellOperator
            src = u
            for i, (a, b) in enumerate(zip(RK_A, RK_B)):
                dst = u if i == len(RK_A) - 1 else (self._alt if i % 2 == 0 else self._alt2)
                self._stage(src, dst, a, b, dt)
                src = dst
        return u

    def rhs_padded(self, u, out=None):
        out = self.op.empty_state() if out is None else out
        self.exchange(u)
        return self.op.rhs_padded(u, out)

    def field_energy(self, u) -> float:
        import torch.distributed as dist

        m = self.op.material
        t = self.op.mass_norm(u, m.permittivity, m.permeability)
        if dist.is_initialized() and dist.get_world_size() > 1:
            dist.all_reduce(t)
        return 0.5 * float(t.item())
