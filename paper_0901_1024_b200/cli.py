"""Command line: ``simulate`` and ``convergence`` on the B200 backend.

Mirrors the two solver subcommands of ``simtdg.cli`` (cli.py:179-200, 270-325,
348-411) with ``--backend b200``: same arguments, same JSON / CSV outputs
(``%.17g`` floats), same ``{"error", "message"}`` JSON on stderr and exit
code 1 for any failure.  ``tune`` and ``layout-stats`` drive the reference's
GT200 emulator and have no B200 counterpart (out of scope).

    python -m paper_0901_1024_b200.cli simulate --order 4 --cells 4 --final-time 0.1
    python -m paper_0901_1024_b200.cli convergence --orders 1,2,3,4 --resolutions 2,3,4
"""

from __future__ import annotations

import argparse
import io
import json
import sys

import numpy as np

_FLOAT_FMT = "%.17g"


def _fmt(value) -> str:
    return _FLOAT_FMT % value if isinstance(value, float) else str(value)


def rows_to_csv(rows: list[dict]) -> str:
    """CSV text with the reference's float format (cli.py:34-58)."""
    import csv

    buf = io.StringIO()
    if rows:
        writer = csv.DictWriter(buf, fieldnames=list(rows[0].keys()), lineterminator="\n")
        writer.writeheader()
        for row in rows:
            writer.writerow({k: _fmt(v) for k, v in row.items()})
    return buf.getvalue()


def fit_eoc(mesh_sizes, errors) -> float:
    """Least-squares slope of log error against log mesh size (cli.py:165-170)."""
    slope, _ = np.polyfit(np.log(np.asarray(mesh_sizes, float)), np.log(np.asarray(errors, float)), 1)
    return float(slope)


def cmd_convergence(orders, resolutions, extent=(1.0, 1.0, 1.0), mode_numbers=(1, 1, 1), final_time=0.75,
                    cfl=1.0, backend="b200", dtype=None) -> list[dict]:
    """Error rows per (order, resolution) plus one fitted-order row each (cli.py:179-200)."""
    from .driver import run_cavity

    rows = []
    for order in orders:
        sizes, errors = [], []
        for m in resolutions:
            run = run_cavity(order, (m, m, m), extent, mode_numbers, final_time, cfl, backend, dtype=dtype)
            sizes.append(run.mesh_size)
            errors.append(run.l2_error)
            rows.append({"row": "error", "order": order, "mesh_size": run.mesh_size,
                         "num_elements": run.num_elements, "l2_error": run.l2_error, "eoc": ""})
        rows.append({"row": "eoc", "order": order, "mesh_size": "", "num_elements": "", "l2_error": "",
                     "eoc": fit_eoc(sizes, errors)})
    return rows


def _triple(text, kind=int):
    parts = [kind(p) for p in str(text).split(",") if p]
    if len(parts) == 1:
        parts = parts * 3
    if len(parts) != 3:
        raise argparse.ArgumentTypeError(f"expected 1 or 3 comma-separated values, got {text!r}")
    return tuple(parts)


def _ints(text):
    return [int(p) for p in str(text).split(",") if p]


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_0901_1024_b200", description="DG Maxwell cavity solver on B200")
    sub = parser.add_subparsers(dest="command", required=True)
    dtypes = ("f32", "f64")

    conv = sub.add_parser("convergence", help="cavity error sweep with fitted orders")
    conv.add_argument("--orders", default="1,2,3,4")
    conv.add_argument("--resolutions", default="2,3,4")
    conv.add_argument("--extent", type=lambda s: _triple(s, float), default=(1.0, 1.0, 1.0))
    conv.add_argument("--mode", type=_triple, default=(1, 1, 1))
    conv.add_argument("--final-time", type=float, default=0.75)
    conv.add_argument("--cfl", type=float, default=1.0)
    conv.add_argument("--backend", choices=("b200",), default="b200")
    conv.add_argument("--dtype", choices=dtypes, default="f64")
    conv.add_argument("--out", default="-")

    sim = sub.add_parser("simulate", help="single cavity run")
    sim.add_argument("--order", type=int, default=3)
    sim.add_argument("--cells", type=_triple, default=(2, 2, 2))
    sim.add_argument("--extent", type=lambda s: _triple(s, float), default=(1.0, 1.0, 1.0))
    sim.add_argument("--mode", type=_triple, default=(1, 1, 1))
    sim.add_argument("--final-time", type=float, default=0.75)
    sim.add_argument("--cfl", type=float, default=1.0)
    sim.add_argument("--backend", choices=("b200",), default="b200")
    sim.add_argument("--dtype", choices=dtypes, default="f32")
    sim.add_argument("--node-file", default=None, help="TetGen .node file (mesh of the same box as --extent)")
    sim.add_argument("--ele-file", default=None, help="TetGen .ele file")
    sim.add_argument("--energy-out", default=None, help="optional energy-trace CSV path")
    sim.add_argument("--out", default="-")
    return parser


def _emit(path: str, text: str) -> None:
    if path == "-":
        sys.stdout.write(text)
    else:
        with open(path, "w") as f:
            f.write(text)


def main(argv=None) -> int:
    parser = _build_parser()
    args = parser.parse_args(argv)
    try:
        import torch

        dtype = torch.float64 if args.dtype == "f64" else torch.float32
        if args.command == "convergence":
            rows = cmd_convergence(_ints(args.orders), _ints(args.resolutions), args.extent, args.mode,
                                   args.final_time, args.cfl, args.backend, dtype=dtype)
            _emit(args.out, rows_to_csv(rows))
        else:
            from .driver import run_cavity
            from .mesh import read_tetgen

            mesh = None
            if (args.node_file is None) != (args.ele_file is None):
                raise ValueError("--node-file and --ele-file must be given together")
            if args.node_file:
                with open(args.node_file) as nf, open(args.ele_file) as ef:
                    mesh = read_tetgen(nf.read(), ef.read())
            run = run_cavity(args.order, args.cells, args.extent, args.mode, args.final_time, args.cfl,
                             args.backend, collect_energy=args.energy_out is not None, mesh=mesh, dtype=dtype)
            if args.energy_out:
                _emit(args.energy_out, rows_to_csv([{"time": t, "energy": e} for t, e in run.energy_trace]))
            summary = {"order": run.order, "num_elements": run.num_elements, "mesh_size": run.mesh_size,
                       "dt": run.dt, "num_steps": run.num_steps, "final_time": run.final_time,
                       "l2_error": run.l2_error, "initial_energy": run.initial_energy,
                       "final_energy": run.final_energy, "max_energy_growth": run.max_energy_growth,
                       "stage_stats": run.stage_stats}
            _emit(args.out, json.dumps(summary, indent=2, sort_keys=True) + "\n")
    except Exception as exc:  # process boundary: JSON error on stderr, rc 1 (cli.py:408-411)
        sys.stderr.write(json.dumps({"error": type(exc).__name__, "message": str(exc)}) + "\n")
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
