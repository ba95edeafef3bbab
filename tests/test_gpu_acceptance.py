"""The reference's solver acceptance criteria (pkg/tests/test_acceptance.py) on the B200 backend.

Criterion 1 (test_acceptance.py:37-52): fitted EOC in [N + 0.5, N + 1.7] for
N = 1..4 on the same cavity runs (final_time 0.75, cfl 1), energy never grows.
Criterion 6 (test_acceptance.py:177-200): 1000 steps at default CFL with
non-increasing energy (per-step relative tolerance 1e-12 in fp64; fp32
adds its rounding, 1e-6) and under 1 % total decay.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_0901_1024_b200 import (CavityMode, build_b200_operator, build_reference_element,  # noqa: E402
                                  generate_box_mesh, map_nodes, run_cavity, stable_dt)
from paper_0901_1024_b200.cli import cmd_convergence, fit_eoc, main  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("order,resolutions", [(1, (4, 6, 8)), (2, (3, 4, 6)), (3, (2, 3, 4)), (4, (2, 3))])
def test_criterion_1_convergence_orders(order, resolutions):
    sizes, errors = [], []
    for m in resolutions:
        run = run_cavity(order, (m, m, m), final_time=0.75, cfl=1.0, dtype=torch.float64)
        assert run.max_energy_growth <= 1e-12
        sizes.append(run.mesh_size)
        errors.append(run.l2_error)
    eoc = fit_eoc(sizes, errors)
    print(f"N={order}: EOC={eoc:.2f} errors={errors}")
    assert order + 0.5 <= eoc <= order + 1.7, (order, eoc)


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 1e-6)])
@pytest.mark.parametrize("order,cells", [(3, 4), (4, 3)])
def test_criterion_6_energy_dissipation(order, cells, dtype, tol):
    mesh = generate_box_mesh((1.0, 1.0, 1.0), (cells,) * 3)
    elem = build_reference_element(order)
    op = build_b200_operator(mesh, elem, dtype=dtype)
    dt = stable_dt(mesh, op.geometry, order, cfl=1.0)
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    energies = torch.zeros(1001, dtype=torch.float64, device=op.device)
    op.mass_norm(u, out=energies[0:1])
    for n in range(1, 1001):
        op.step(u, dt)
        op.mass_norm(u, out=energies[n:n + 1])
    e = energies.cpu().numpy()
    assert np.all(e[1:] <= e[:-1] * (1.0 + tol))
    decay = 1.0 - e[-1] / e[0]
    print(f"N={order} K={mesh.num_elements} {dtype}: decay {decay * 100:.4f}%")
    assert 0.0 <= decay < 0.01


def test_cli_convergence_and_simulate(tmp_path, capsys):
    rows = cmd_convergence([2], [2, 3], final_time=0.1)
    assert [r["row"] for r in rows] == ["error", "error", "eoc"]
    assert math.isfinite(rows[-1]["eoc"])
    energy_csv = tmp_path / "energy.csv"
    assert main(["simulate", "--order", "2", "--cells", "2", "--final-time", "0.05",
                 "--energy-out", str(energy_csv)]) == 0
    out = capsys.readouterr().out
    import json

    summary = json.loads(out)
    assert summary["num_elements"] == 48 and summary["max_energy_growth"] <= 1e-6
    lines = energy_csv.read_text().splitlines()
    assert lines[0] == "time,energy" and len(lines) == summary["num_steps"] + 2
