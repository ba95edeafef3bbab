"""Loose performance guards (a regression of several x fails; the numbers themselves live in bench.py).

C1 through the CUDA-graph path (launch-bound) and the fp64 kernel at 48k tets; bounds
are ~3x the round-2 measurements (C1 14.7 us, fp64 N=4 at 48k ~0.2 ms per stage).
"""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_0901_1024_b200 import (CavityMode, build_b200_operator, build_reference_element,  # noqa: E402
                                  generate_box_mesh, map_nodes, stable_dt)


def _us_per_stage(cells, order, dtype, steps, graph):
    torch.cuda.set_device(0)
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    elem = build_reference_element(order)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    dt = stable_dt(mesh, op.geometry, order)
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    op.advance(u, dt, 8, use_graph=graph)
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        op.advance(u, dt, steps, use_graph=graph)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / (5 * steps)
        best = us if best is None else min(best, us)
    return best


def test_c1_graph_path_stage_time():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    us = _us_per_stage((6, 6, 7), 3, torch.float32, 64, True)
    print(f"C1 {us:.1f} us per stage")
    assert us < 45.0


def test_fp64_stage_time():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    us = _us_per_stage((20, 20, 20), 4, torch.float64, 10, False)
    print(f"fp64 N=4 48k {us:.1f} us per stage")
    assert us < 700.0
