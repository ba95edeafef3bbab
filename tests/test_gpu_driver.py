"""run_cavity(backend="b200") against the reference driver loop (cli.py:81-164) restated on the oracle."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import build_oracle_operator, rk4_step  # noqa: E402
from paper_0901_1024_b200 import (CavityMode, UnstableRunError, build_reference_element,  # noqa: E402
                                  compute_geometry, field_energy, generate_box_mesh, l2_error, map_nodes,
                                  run_cavity, stable_dt)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _reference_loop(order, cells, final_time):
    """The reference's run_cavity loop (cli.py:99-164) with the oracle RHS, fp64 on the host."""
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    elem = build_reference_element(order)
    geo = compute_geometry(mesh)
    nodes = map_nodes(mesh, elem)
    mode = CavityMode(1, 1, 1, (1.0, 1.0, 1.0))
    ora = build_oracle_operator(mesh, elem)
    dt = stable_dt(mesh, geo, order)
    n = max(1, math.ceil(final_time / dt))
    dt = final_time / n
    u = mode.evaluate(nodes, 0.0)
    energies = [field_energy(u, elem, geo)]
    for _ in range(n):
        u = rk4_step(u, 0.0, dt, lambda t, y: ora.rhs(y))
        energies.append(field_energy(u, elem, geo))
    return n, dt, energies, l2_error(u, mode, final_time, elem, geo, nodes)


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-10), (torch.float32, 1e-5)])
def test_run_cavity_matches_reference_loop(dtype, tol):
    order, cells, final_time = 3, (2, 2, 2), 0.05
    n, dt, energies, err = _reference_loop(order, cells, final_time)
    run = run_cavity(order, cells, final_time=final_time, collect_energy=True, dtype=dtype, check_every=7)
    assert run.num_steps == n and math.isclose(run.dt, dt, rel_tol=1e-15)
    assert run.num_elements == 48
    got = np.array([e for _, e in run.energy_trace])
    assert len(got) == n + 1
    assert np.max(np.abs(got - energies) / energies[0]) < tol
    assert abs(run.l2_error - err) <= tol * max(err, 1e-3) + 1e-7
    assert run.max_energy_growth <= 1e-6
    assert math.isclose(run.final_time, final_time, rel_tol=1e-12)
    st = run.stage_stats["lsrk_stage"]  # per-kernel device time (pipeline.py stage_stats counterpart)
    assert st["launches"] == 5 * n and st["ms"] > 0.0


def test_run_cavity_errors():
    with pytest.raises(ValueError):
        run_cavity(2, (1, 1, 1), backend="emulated")
    with pytest.raises(UnstableRunError):
        run_cavity(2, (1, 1, 1), final_time=0.05, blowup_factor=-1.0)
