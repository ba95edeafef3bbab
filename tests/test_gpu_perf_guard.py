"""Loose performance guards (a regression of several x fails; the numbers themselves live in bench.py).

C1 through the CUDA-graph path (launch-bound), the fp64 kernel and the tensor kernels'
lane mappings at 48k tets; bounds are ~3x the round-2 measurements (C1 6.9-7.7 us, fp64
N=4 at 48k 0.2 ms per stage).
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


@pytest.mark.parametrize("order,bound_us", [(4, 250.0), (5, 420.0), (7, 1150.0), (9, 2450.0)])
def test_tensor_stage_time(order, bound_us):
    """The tensor kernels per lane mapping (N=4 MAP 0 two CTAs/SM, N=5 / 7 the 42-element three-component
    tiles, N=9 the 21-element tile) at 48k tets: ~3x the round-2 stage times (79 / 139 / 384 / 818 us)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    us = _us_per_stage((20, 20, 20), order, torch.float32, 6, False)
    print(f"tensor N={order} 48k {us:.1f} us per stage")
    assert us < bound_us
