"""Cavity driver with the B200 backend: the reference's ``run_cavity`` loop, device-resident.

Mirrors ``simtdg.cli.run_cavity`` (cli.py:81-164): box mesh (or a given
mesh), TM cavity mode as initial state, ``dt = stable_dt`` rounded so that
``final_time`` is hit exactly (cli.py:121-123), one LSRK4 step per iteration,
``field_energy`` after every step with the blow-up check (cli.py:132-144),
``l2_error`` at the end.  The state never leaves HBM: each step is the fused
stage kernel x5 and the energy is a device reduction written into a
preallocated slot, so the host synchronises only every ``check_every`` steps
(the blow-up check still reports the first offending step, as the reference).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .maxwell import VACUUM, CavityMode, Material, stable_dt
from .mesh import generate_box_mesh
from .refelem import build_reference_element

BACKENDS = ("b200",)


class UnstableRunError(RuntimeError):
    """The solver blew up (energy grew far beyond its initial value) -- cli.py:30-31."""


@dataclass
class CavityRun:
    """Same fields as the reference's CavityRun (cli.py:64-78)."""

    order: int
    num_elements: int
    mesh_size: float
    dt: float
    num_steps: int
    final_time: float
    l2_error: float
    initial_energy: float
    final_energy: float
    max_energy_growth: float
    energy_trace: list = field(default_factory=list)
    stage_stats: dict = field(default_factory=dict)


def run_cavity(order: int, cells, extent=(1.0, 1.0, 1.0), mode_numbers=(1, 1, 1), final_time: float = 0.75,
               cfl: float = 1.0, backend: str = "b200", material: Material = VACUUM,
               collect_energy: bool = False, blowup_factor: float = 1e3, mesh=None, *,
               dtype=None, device=None, check_every: int = 64) -> CavityRun:
    """Integrate one cavity eigenmode on the GPU and measure the error against it (cli.py:81-164)."""
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}")
    import torch

    from .operator import build_b200_operator

    dtype = torch.float32 if dtype is None else dtype
    if mesh is None:
        mesh = generate_box_mesh(extent, cells)
    elem = build_reference_element(order)
    mode = CavityMode(*mode_numbers, extent=tuple(float(x) for x in extent), material=material)
    op = build_b200_operator(mesh, elem, material, dtype=dtype, device=device)
    geo, nodes = op.geometry, op.nodes

    dt = stable_dt(mesh, geo, order, material, cfl)
    num_steps = max(1, math.ceil(final_time / dt))
    dt = final_time / num_steps

    u = op.to_padded(mode.evaluate(nodes, 0.0))
    weights = (material.permittivity, material.permeability)
    energies = torch.zeros(num_steps + 1, dtype=torch.float64, device=op.device)
    op.mass_norm(u, *weights, out=energies[0:1])
    e0 = 0.5 * float(energies[0].item())

    t = 0.0
    checked = 0
    e_prev = e0
    max_growth = 0.0
    trace = [(0.0, e0)] if collect_energy else []

    def scan(upto: int) -> None:
        nonlocal checked, e_prev, max_growth
        vals = (0.5 * energies[checked + 1:upto + 1]).cpu().numpy()
        for i, energy in enumerate(vals):
            step = checked + 1 + i
            energy = float(energy)
            if e_prev > 0.0:
                max_growth = max(max_growth, (energy - e_prev) / e_prev)
            if not energy <= blowup_factor * e0:  # NaN counts as a blow-up
                raise UnstableRunError(
                    f"energy grew to {energy / e0:.1f}x its initial value at t={step * dt:.4g}")
            e_prev = energy
            if collect_energy:
                trace.append((step * dt, energy))
        checked = upto

    op.collect_stats = True  # per-kernel device time -> CavityRun.stage_stats
    for n in range(1, num_steps + 1):
        op.step(u, dt)
        t += dt
        op.mass_norm(u, *weights, out=energies[n:n + 1])
        if n % check_every == 0 or n == num_steps:
            scan(n)

    edges = mesh.vertices[mesh.elements]
    h = max(float(np.linalg.norm(edges[:, a] - edges[:, b], axis=1).max())
            for a in range(4) for b in range(a + 1, 4))
    return CavityRun(order=order, num_elements=mesh.num_elements, mesh_size=h, dt=dt, num_steps=num_steps,
                     final_time=t, l2_error=op.l2_error(u, mode, t), initial_energy=e0, final_energy=e_prev,
                     max_energy_growth=max_growth, energy_trace=trace,
                     stage_stats={k: v.to_dict() for k, v in op.stage_stats.items()})
