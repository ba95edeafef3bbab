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
