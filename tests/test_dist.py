"""Multi-GPU partition and halo plan, checked on CPU with torch.distributed gloo.

The GPU path (DistributedMaxwellOperator) packs the face traces of the cut
faces (dgm_trace_pack: 6 x Nfp values per (element, face) pair), exchanges
them with NCCL send/recv and scatters them into the face nodes of the ghost
rows (dgm_trace_unpack).  Here the same trace lists drive a CPU exchange over
gloo (numpy gathers / scatters with the kernels' semantics; ghost nodes off
the cut faces stay zero), each rank evaluates the RHS of its owned elements
with the CPU oracle on its sub-mesh, and the distributed LSRK4 run must equal
the single-process oracle run.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import OracleOperator
from oracle.dg_oracle import RK_A, RK_B
from paper_0901_1024_b200 import build_reference_element, generate_box_mesh
from paper_0901_1024_b200.dist import build_box_domain, build_mesh_domain, split_range
from paper_0901_1024_b200.facemaps import build_face_maps

EXTENT = (1.0, 0.8, 0.9)
CELLS = (6, 2, 2)


def _global_view(dom):
    """Local (owned + ghost) neighbor ids mapped back to global ids."""
    g0 = dom.owned[0]
    ids = np.concatenate([np.arange(g0, dom.owned[1]), dom.ghost_global])
    nb = ids[dom.maps.neighbors.astype(np.int64)]
    return nb


@pytest.mark.parametrize("world", [1, 2, 3, 6])
@pytest.mark.parametrize("order", [1, 3])
def test_box_domains_reproduce_global_maps(world, order):
    elem = build_reference_element(order)
    mesh = generate_box_mesh(EXTENT, CELLS)
    gmaps = build_face_maps(mesh, elem)
    doms = [build_box_domain(EXTENT, CELLS, elem, r, world) for r in range(world)]
    covered = []
    for dom in doms:
        g0, g1 = dom.owned
        covered.append((g0, g1))
        assert np.array_equal(_global_view(dom), np.where(gmaps.codes[g0:g1] >= 0, gmaps.neighbors[g0:g1],
                                                          np.arange(g0, g1)[:, None]))
        # the reference's plus-side node ids, through the rank's own code table
        inner = dom.maps.codes >= 0
        loc = dom.maps.code_table[np.where(inner, dom.maps.codes, 0)]
        glo = gmaps.code_table[np.where(gmaps.codes[g0:g1] >= 0, gmaps.codes[g0:g1], 0)]
        assert np.array_equal(loc[inner], glo[inner])
        assert np.array_equal(dom.maps.codes < 0, gmaps.codes[g0:g1] < 0)
        p, q = dom.interior
        assert (dom.maps.neighbors[p:q][dom.maps.codes[p:q] >= 0] < dom.num_owned).all()
        mdom = build_mesh_domain(mesh, elem, dom.rank, world, gmaps)
        assert mdom.owned == dom.owned
        assert np.array_equal(mdom.ghost_global, dom.ghost_global)
        assert {k: v.tolist() for k, v in mdom.send.items()} == {k: v.tolist() for k, v in dom.send.items()}
        assert mdom.recv == dom.recv
        assert np.allclose(mdom.geo_words, dom.geo_words, rtol=0, atol=1e-15)
    assert covered[0][0] == 0 and covered[-1][1] == mesh.num_elements
    assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
    # send/recv symmetry: what r sends to q is exactly q's ghost block from r, in order
    for r, dr in enumerate(doms):
        for q, ids in dr.send.items():
            begin, cnt = doms[q].recv[r]
            k_own = doms[q].num_owned
            want = doms[q].ghost_global[begin - k_own:begin - k_own + cnt]
            assert np.array_equal(ids.astype(np.int64) + dr.owned[0], want)
    # face traces: r's send list to q and q's receive list from r name the same (global element,
    # face) pairs in the same order; each is a cut face (the neighbour across it is on the other rank)
    for r, dr in enumerate(doms):
        assert set(dr.send_traces) == set(dr.send) and set(dr.recv_traces) == set(dr.recv)
        for q, tr in dr.send_traces.items():
            sent = np.stack([tr[:, 0].astype(np.int64) + dr.owned[0], tr[:, 1]], 1)
            rt = doms[q].recv_traces[r]
            got = np.stack([doms[q].ghost_global[rt[:, 0] - doms[q].num_owned], rt[:, 1]], 1)
            assert np.array_equal(sent, got)
            across = gmaps.neighbors[sent[:, 0], sent[:, 1]]
            q0, q1 = doms[q].owned
            assert ((across >= q0) & (across < q1)).all() and (gmaps.codes[sent[:, 0], sent[:, 1]] >= 0).all()
            # every (owned element, face) of r glued to q's range is listed exactly once
            g0, g1 = dr.owned
            nb, cd = gmaps.neighbors[g0:g1], gmaps.codes[g0:g1]
            assert len(tr) == int(((cd >= 0) & (nb >= q0) & (nb < q1)).sum())
        mdom = build_mesh_domain(mesh, elem, r, world, gmaps)
        for q, tr in dr.send_traces.items():
            assert np.array_equal(mdom.send_traces[q], tr) and np.array_equal(mdom.recv_traces[q], dr.recv_traces[q])


def test_split_range_balanced():
    parts = [split_range(10, 3, r) for r in range(3)]
    assert parts == [(0, 4), (4, 7), (7, 10)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(dom, ext: torch.Tensor):
    """Fill the cut-face nodes of ext's ghost rows from their owners (CPU/gloo stand-in for
    dgm_trace_pack / dgm_trace_unpack + NCCL): buffer[c][field][i] = u[field][elem][fmask[face][i]]."""
    fmask = np.asarray(dom.elem.face_nodes)
    x = ext.numpy()
    reqs, bufs = [], {}
    for peer, tr in dom.send_traces.items():
        e, f = tr[:, 0].astype(np.int64), tr[:, 1].astype(np.int64)
        buf = torch.from_numpy(np.ascontiguousarray(x[:, e[:, None], fmask[f]].transpose(1, 0, 2)))
        reqs.append(dist.isend(buf, peer))
        bufs[("s", peer)] = buf
    for peer, tr in dom.recv_traces.items():
        buf = torch.empty((len(tr), 6, fmask.shape[1]), dtype=ext.dtype)
        reqs.append(dist.irecv(buf, peer))
        bufs[("r", peer)] = buf
    for r in reqs:
        r.wait()
    for peer, tr in dom.recv_traces.items():
        e, f = tr[:, 0].astype(np.int64), tr[:, 1].astype(np.int64)
        x[:, e[:, None], fmask[f]] = bufs[("r", peer)].numpy().transpose(1, 0, 2)


def _worker(rank, world, port, order, steps, dt, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        elem = build_reference_element(order)
        dom = build_box_domain(EXTENT, CELLS, elem, rank, world)
        sub = dom.mesh
        ora = OracleOperator(sub.vertices, sub.elements, elem)
        n_p = elem.num_nodes
        g0, g1 = dom.owned
        rng = np.random.default_rng(7)
        k_glob = CELLS[0] * CELLS[1] * CELLS[2] * 6
        u_glob0 = rng.normal(size=(6, k_glob, n_p))
        # local state: owned rows then ghost rows (ghosts filled only by exchange)
        ext = torch.zeros((6, dom.num_owned + dom.num_ghost, n_p), dtype=torch.float64)
        ext[:, :dom.num_owned] = torch.from_numpy(u_glob0[:, g0:g1])
        # local slot of every sub-mesh element (-1: not present locally)
        sub_ids = np.arange(sub.num_elements) + dom.sub_offset
        slot = np.full(sub.num_elements, -1)
        own = (sub_ids >= g0) & (sub_ids < g1)
        slot[own] = sub_ids[own] - g0
        gpos = np.searchsorted(dom.ghost_global, sub_ids)
        is_ghost = ~own & (gpos < dom.num_ghost)
        is_ghost[is_ghost] &= dom.ghost_global[gpos[is_ghost]] == sub_ids[is_ghost]
        slot[is_ghost] = dom.num_owned + gpos[is_ghost]

        def local_rhs(x: torch.Tensor) -> np.ndarray:
            _exchange(dom, x)
            full = np.zeros((6, sub.num_elements, n_p))
            present = slot >= 0
            full[:, present] = x.numpy()[:, slot[present]]
            return ora.rhs(full)[:, own]

        res = torch.zeros((6, dom.num_owned, n_p), dtype=torch.float64)
        for _ in range(steps):
            for a, b in zip(RK_A, RK_B):
                k = torch.from_numpy(local_rhs(ext))
                res = a * res + dt * k
                ext[:, :dom.num_owned] += b * res
        out_q.put((rank, g0, g1, ext[:, :dom.num_owned].numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_distributed_lsrk_matches_single_process(world):
    order, steps, dt = 2, 2, 2e-3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, order, steps, dt, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    elem = build_reference_element(order)
    mesh = generate_box_mesh(EXTENT, CELLS)
    ora = OracleOperator(mesh.vertices, mesh.elements, elem)
    u = np.random.default_rng(7).normal(size=(6, mesh.num_elements, elem.num_nodes))
    res = np.zeros_like(u)
    for _ in range(steps):
        for a, b in zip(RK_A, RK_B):
            res = a * res + dt * ora.rhs(u)
            u = u + b * res
    got = np.zeros_like(u)
    for _, g0, g1, block in parts:
        got[:, g0:g1] = block
    assert np.abs(got - u).max() <= 1e-12 * np.abs(u).max()


def test_interior_locality_order_keeps_boundary_and_ghost_slots():
    """DistributedMaxwellOperator's locality order permutes only the interior range."""
    from paper_0901_1024_b200.dist import DistributedMaxwellOperator
    from paper_0901_1024_b200.ordering import permute_maps

    elem = build_reference_element(3)
    dom = build_box_domain((2.0, 1.0, 1.0), (12, 4, 4), elem, 0, 2)
    order = DistributedMaxwellOperator._interior_order(dom)
    k = dom.num_owned
    p, q = dom.interior
    assert q - p > 64 and np.array_equal(np.sort(order), np.arange(k))
    assert np.array_equal(order[:p], np.arange(p)) and np.array_equal(order[q:], np.arange(q, k))
    assert not np.array_equal(order[p:q], np.arange(p, q))
    pm = permute_maps(dom.maps, order)
    ghost = dom.maps.neighbors >= k
    assert np.array_equal(pm.neighbors[ghost[order]], dom.maps.neighbors[order][ghost[order]])
    inner = (pm.codes >= 0) & (pm.neighbors < k)
    assert np.array_equal(order[pm.neighbors[inner]], dom.maps.neighbors[order][inner])
    for ids in dom.send.values():  # every sent row is outside the permuted range
        assert np.all((ids < p) | (ids >= q))
