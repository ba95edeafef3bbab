"""GPU check of the partitioned operator on one device: several in-process ranks.

Exercises the real dgm_halo_pack / dgm_halo_unpack kernels, the ghost-slot
layout (field_stride = owned + ghosts) and the interior/boundary launch split;
the NCCL transfer is replaced by device copies between the ranks' buffers
(multi-process NCCL needs one GPU per rank; the plans are covered by the gloo
tests in test_dist.py).
"""

import numpy as np
import pytest
from conftest import rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_0901_1024_b200 import build_b200_operator, build_reference_element, generate_box_mesh  # noqa: E402
from paper_0901_1024_b200.dist import DistributedMaxwellOperator, build_box_domain  # noqa: E402
from paper_0901_1024_b200.stepper import RK_A, RK_B  # noqa: E402

EXTENT = (1.0, 0.9, 0.8)
CELLS = (6, 3, 2)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_in_process_ranks_match_single_operator(world, dtype):
    order, dt, steps = 3, 1e-3, 2
    elem = build_reference_element(order)
    mesh = generate_box_mesh(EXTENT, CELLS)
    u0 = np.random.default_rng(4).normal(size=(6, mesh.num_elements, elem.num_nodes))
    single = build_b200_operator(mesh, elem, dtype=dtype)
    ref = single.to_padded(u0)
    single.advance(ref, dt, steps, use_graph=False)
    want = single.from_padded(ref).cpu().numpy()

    ranks = []
    for r in range(world):
        dom = build_box_domain(EXTENT, CELLS, elem, r, world)
        dop = DistributedMaxwellOperator(dom, dtype=dtype)
        g0, g1 = dom.owned
        u = dop.op.to_padded(u0[:, g0:g1])  # owned rows packed; ghost slots zero until exchanged
        ranks.append({"dop": dop, "cur": u, "nxt": dop.op.empty_state(), "res": dop.op.empty_state()})

    for _ in range(steps):
        for a, b in zip(RK_A, RK_B):
            sends = [rk["dop"].pack(rk["cur"]) for rk in ranks]
            for r, rk in enumerate(ranks):
                for peer, buf in rk["dop"].recv_buffers.items():
                    buf.copy_(sends[peer][r])
            for rk in ranks:
                rk["dop"].unpack(rk["cur"])
            for rk in ranks:
                (p, q), boundary = rk["dop"].stage_ranges()
                for lo, hi in [(p, q)] + boundary:
                    if hi > lo:
                        rk["dop"].op.lsrk_stage(rk["cur"], rk["nxt"], rk["res"], a, b, dt, lo, hi)
                rk["cur"], rk["nxt"] = rk["nxt"], rk["cur"]
    got = np.zeros_like(want)
    for rk in ranks:
        g0, g1 = rk["dop"].domain.owned
        got[:, g0:g1] = rk["dop"].op.from_padded(rk["cur"]).cpu().numpy()
    tol = 1e-6 if dtype == torch.float32 else 1e-13
    assert rel_l2(got, want) < tol
    # every rank really had ghosts and an interior range
    for rk in ranks:
        d = rk["dop"].domain
        assert d.num_ghost > 0 and d.interior[1] > d.interior[0]


class _DeviceMailbox:
    """In-process stand-in for NCCL send/recv between ranks running in threads of one process.

    isend snapshots the buffer on the sender's current (communication) stream and posts it with an
    event; irecv takes the matching post, makes the receiver's current stream wait for the event and
    copies.  So DistributedMaxwellOperator._exchange_async / _stage / advance run unmodified, with
    their real communication stream, events and buffer reuse across stages.
    """

    def __init__(self):
        import queue
        import threading
        from collections import defaultdict

        self.posts = defaultdict(queue.Queue)
        self.local = threading.local()
        self.calls = 0

    @staticmethod
    def isend(*a, **k):  # markers only (P2POp below records which one was passed)
        raise AssertionError("not called directly")

    @staticmethod
    def irecv(*a, **k):
        raise AssertionError("not called directly")

    def P2POp(self, op, tensor, peer, group=None, tag=0):  # noqa: N802 (torch name)
        return (op, tensor, peer)

    def batch_isend_irecv(self, ops):
        me = self.local.rank
        stream = torch.cuda.current_stream()
        self.calls += 1
        for op, t, peer in ops:
            if op is self.isend:
                snap = t.clone()
                ev = torch.cuda.Event()
                ev.record(stream)
                self.posts[(me, peer)].put((snap, ev))
        for op, t, peer in ops:
            if op is self.irecv:
                snap, ev = self.posts[(peer, me)].get(timeout=120)
                stream.wait_event(ev)
                snap.record_stream(stream)
                t.copy_(snap)

        class _Done:
            def wait(self):
                return True

        return [_Done()]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dtype,order", [(torch.float32, 4), (torch.float64, 3)])
def test_distributed_advance_through_device_transport(monkeypatch, world, dtype, order):
    """DistributedMaxwellOperator.advance itself (comm stream, face-trace pack / exchange / unpack
    overlapped with the interior launch) on in-process ranks in threads == the single operator."""
    import threading

    import torch.distributed as dist

    dt, steps = 1e-3, 3
    extent, cells = (1.5, 0.9, 0.8), (9, 4, 3)
    elem = build_reference_element(order)
    mesh = generate_box_mesh(extent, cells)
    u0 = np.random.default_rng(11).normal(size=(6, mesh.num_elements, elem.num_nodes))
    single = build_b200_operator(mesh, elem, dtype=dtype)
    ref = single.to_padded(u0)
    single.advance(ref, dt, steps, use_graph=False)
    want = single.from_padded(ref).cpu().numpy()

    box = _DeviceMailbox()
    for name in ("P2POp", "isend", "irecv", "batch_isend_irecv"):
        monkeypatch.setattr(dist, name, getattr(box, name))
    doms = [build_box_domain(extent, cells, elem, r, world) for r in range(world)]
    ops = [DistributedMaxwellOperator(d, dtype=dtype) for d in doms]
    # the halo is face traces: 6 x Nfp values per cut face
    for d, o in zip(doms, ops):
        for peer, buf in o.recv_buffers.items():
            assert buf.shape == (len(d.recv_traces[peer]), 6 * elem.num_face_nodes)
    states = [o.to_padded(u0[:, d.owned[0]:d.owned[1]]) for d, o in zip(doms, ops)]
    errors = []

    def run(r):
        try:
            torch.cuda.set_device(0)
            box.local.rank = r
            ops[r].advance(states[r], dt, steps)
            torch.cuda.synchronize()
        except Exception as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    assert box.calls == world * steps * 5
    got = np.zeros_like(want)
    for d, o, s in zip(doms, ops, states):
        got[:, d.owned[0]:d.owned[1]] = o.op.from_padded(s).cpu().numpy()
    tol = 1e-6 if dtype == torch.float32 else 1e-13
    err = rel_l2(got, want)
    print(f"world={world} {dtype} N={order}: rel L2 {err:.2e}")
    assert err < tol


def _nccl_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        extent, cells, order, dt, steps = (1.5, 0.9, 0.8), (9, 4, 3), 4, 1e-3, 3
        elem = build_reference_element(order)
        mesh = generate_box_mesh(extent, cells)
        u0 = np.random.default_rng(11).normal(size=(6, mesh.num_elements, elem.num_nodes))
        dom = build_box_domain(extent, cells, elem, rank, world)
        dop = DistributedMaxwellOperator(dom, dtype=torch.float32, device=f"cuda:{rank}")
        u = dop.to_padded(u0[:, dom.owned[0]:dom.owned[1]])
        dop.advance(u, dt, steps)
        q.put((rank, dom.owned, dop.op.from_padded(u).cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_nccl_two_ranks_match_single_operator():
    """Two processes, one GPU each, NCCL send/recv (runs only where two GPUs are visible)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    extent, cells, order, dt, steps = (1.5, 0.9, 0.8), (9, 4, 3), 4, 1e-3, 3
    elem = build_reference_element(order)
    mesh = generate_box_mesh(extent, cells)
    u0 = np.random.default_rng(11).normal(size=(6, mesh.num_elements, elem.num_nodes))
    single = build_b200_operator(mesh, elem, dtype=torch.float32)
    ref = single.to_padded(u0)
    single.advance(ref, dt, steps, use_graph=False)
    want = single.from_padded(ref).cpu().numpy()
    got = np.zeros_like(want)
    for _, (g0, g1), block in parts:
        got[:, g0:g1] = block
    assert rel_l2(got, want) < 1e-6


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_multi_rank_path_on_one_gpu(scaling):
    """bench.py's N > 1 path end to end (torchrun, 2 ranks, DistributedMaxwellOperator, halo exchange,
    max-over-ranks timing, e2e): both ranks on GPU 0 over gloo (DGM_BENCH_ONE_GPU=1; NCCL refuses two
    ranks on one device).  Checks the JSON line only -- the numbers of a shared GPU mean nothing."""
    import json
    import os
    import socket
    import subprocess
    import sys

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, DGM_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--cells", "12", "10", "10", "--scaling", scaling]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 prints one line
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0 and d["e2e"]["value"] > 0
    k = 12 * 10 * 10 * 6
    assert d["config"]["global_elements"] == (k if scaling == "strong" else 2 * k)
