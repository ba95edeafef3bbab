"""Benchmark of the B200 nodal-DG Maxwell operator (one JSON line on rank 0).

Workload (BASELINE.json configs[2], the metric's N=4 single-GPU config): PEC
cubic cavity, box (55,55,55) -> 998,250 tets, order N=4, fp32, TM (1,1,1)
cavity-mode initial state, dt = stable_dt(cfl=1).  A *step* is one LSRK4
step = 5 launches of the fused stage kernel over all elements.  The state
register (0.86 GB) and residual are far larger than the 126 MB L2, so no
explicit flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 runs under torchrun, one rank per GPU (NCCL); see DESIGN.md.
--impl reference times the reference algorithm (the numpy oracle port of
simtdg's ReferenceMaxwellOperator.rhs + rk4_step) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Maxwell DG net GFLOP/s & DOF-updates/s per RK4 step (N=4, tets); HBM GB/s"
UNIT = "GFLOP/s"
ORDER = 4
CELLS = (55, 55, 55)
CPU_SAMPLE_CELLS = (6, 6, 7)


def _flatten(d, prefix=""):
    for key, val in (d.items() if isinstance(d, dict) else []):
        path = f"{prefix}.{key}" if prefix else str(key)
        if isinstance(val, dict):
            yield from _flatten(val, path)
        elif isinstance(val, (int, float)) and not isinstance(val, bool):
            yield path, float(val)


def _peaks() -> dict:
    """HBM peak for the roofline: MEASURED_PEAKS.json (driver-written) else the B200_PROFILING.md fallback.

    The file's key names are not fixed here, so its numeric entries are searched for an HBM / DRAM
    / copy bandwidth; the sustained figure is preferred (the stage kernel runs inside a long step),
    then burst, then any; values below 100 are taken as TB/s.
    """
    fallback = {"hbm_gbs": 6650.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)", "_fallback": True}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            data = json.load(f)
    except (OSError, ValueError):
        return fallback
    cands = [(k, v) for k, v in _flatten(data)
             if any(t in k.lower() for t in ("hbm", "dram", "copy", "mem_bw", "bandwidth")) and v > 0
             and not any(t in k.lower() for t in ("tflop", "flops", "mhz", "clock"))]
    if not cands:
        return fallback

    def rank(item):
        k = item[0].lower()
        return (0 if "sustain" in k else 1 if "burst" in k else 2, k)

    key, val = sorted(cands, key=rank)[0]
    gbs = val * 1000.0 if val < 100.0 else val
    out = {"hbm_gbs": gbs, "source": f"MEASURED_PEAKS.json {key}"}
    for k, v in _flatten(data):
        if "mhz" in k.lower() and "max" in k.lower():
            out["sm_max_mhz"] = v
    return out


def _ncu_summary() -> dict:
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 100 ms by a background reader.

    Started before the warm-up so the first sample exists before the timed region; every line is
    stamped on arrival and ``summary()`` reports the samples that arrived inside the marked timed
    window (``window: "timed"``), or -- if the timed region was shorter than one sampling period --
    the samples of the whole run (``window: "run"``).
    """

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.samples = []  # (arrival time, line)
        self.t0 = self.t1 = None

    def __enter__(self):
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self

        def reader():
            for line in self.proc.stdout:
                if line.strip():
                    self.samples.append((time.time(), line))

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        deadline = time.time() + 5.0  # wait for the first sample (nvidia-smi start-up)
        while not self.samples and time.time() < deadline:
            time.sleep(0.02)
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_stop(self):
        self.t1 = time.time() + 0.1  # the line reporting the last timed interval arrives a period later

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)

    def summary(self) -> dict:
        lines = [l for t, l in self.samples if self.t0 is not None and self.t0 <= t <= (self.t1 or t)]
        window = "timed"
        if not lines:
            lines, window = [l for _, l in self.samples], "run"
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference_rate(order: int, cells, steps: int, warmup: int = 0):
    """Time the oracle port (reference algorithm, single thread) on a bounded sample."""
    import numpy as np

    from oracle import build_oracle_operator, rk4_step
    from paper_0901_1024_b200 import (CavityMode, build_reference_element, compute_geometry, generate_box_mesh,
                                      map_nodes, stable_dt)
    from paper_0901_1024_b200.perfmodel import flops_per_element_stage

    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    elem = build_reference_element(order)
    ora = build_oracle_operator(mesh, elem)
    u = CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0)
    dt = stable_dt(mesh, compute_geometry(mesh), order)
    for _ in range(warmup):
        u = rk4_step(u, 0.0, dt, lambda t, y: ora.rhs(y))
    t0 = time.perf_counter()
    for _ in range(steps):
        u = rk4_step(u, 0.0, dt, lambda t, y: ora.rhs(y))
    sec = time.perf_counter() - t0
    k = mesh.num_elements
    flops = flops_per_element_stage(order) * k * 5 * steps
    dof = 6 * elem.num_nodes * k * steps
    assert np.isfinite(u).all()
    return {"gflops": flops / sec / 1e9, "dof_updates_per_s": dof / sec, "seconds": sec, "elements": k,
            "steps": steps}


def run_reference(args) -> None:
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    r = cpu_reference_rate(ORDER, CPU_SAMPLE_CELLS, args.steps, args.warmup)
    sample = (f"box {CPU_SAMPLE_CELLS} -> {r['elements']} tets, N={ORDER}, {args.steps} LSRK4 steps after "
              f"{args.warmup} warm-up (the full {CELLS} workload needs ~44 GB and ~7 min per step on this path); "
              "rate is per-DOF and nearly K-independent")
    line = {
        "metric": METRIC, "value": r["gflops"], "unit": UNIT, "impl": "reference", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "dof_updates_per_s": r["dof_updates_per_s"],
        "config": {"workload": f"C3 Maxwell PEC cavity N={ORDER}, box {CELLS}", "order": ORDER,
                   "sample_elements": r["elements"], "path": "oracle port of simtdg ReferenceMaxwellOperator.rhs "
                   "+ rk4_step (numpy einsum, single-threaded as the reference)"},
        "cpu_baseline": {"value": r["gflops"], "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": r["gflops"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args) -> None:
    import numpy as np
    import torch

    from paper_0901_1024_b200 import (CavityMode, build_b200_operator, build_reference_element, compute_geometry,
                                      generate_box_mesh, map_nodes, stable_dt)
    from paper_0901_1024_b200.perfmodel import bytes_per_element_stage, dofs, flops_per_element_stage

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    dtype = torch.float64 if args.dtype == "f64" else torch.float32
    word = 8 if dtype == torch.float64 else 4
    cells = tuple(args.cells)
    t_setup = time.perf_counter()
    elem = build_reference_element(args.order)
    if world == 1:
        mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
        op = build_b200_operator(mesh, elem, dtype=dtype, device=dev, path=args.path,
                                 reorder={"auto": None, "natural": False, "morton": "morton",
                                          "columns": True}[args.element_order],
                                 face_slots=None if args.face_slots == "auto" else False)
        dt = stable_dt(mesh, op.geometry, args.order)
        extent = (1.0, 1.0, 1.0)
        u0_host = CavityMode(1, 1, 1, extent).evaluate(map_nodes(mesh, elem), 0.0)
        runner = op
    else:
        from paper_0901_1024_b200.dist import DistributedMaxwellOperator, build_box_domain
        from paper_0901_1024_b200.mesh import Mesh, compute_geometry as _cg

        # weak scaling: rank r owns cells [r*nx, (r+1)*nx) of a (world*nx, ny, nz) box of extent (world,1,1)
        extent = (float(world), 1.0, 1.0)
        gcells = (cells[0] * world, cells[1], cells[2])
        dom = build_box_domain(extent, gcells, elem, rank, world)
        runner = DistributedMaxwellOperator(dom, dtype=dtype, device=dev, path=args.path,
                                            reorder={"auto": None, "natural": False}.get(args.element_order, True),
                                            face_slots=None if args.face_slots == "auto" else False)
        op = runner.op
        lo = dom.owned[0] - dom.sub_offset
        own_mesh = Mesh(dom.mesh.vertices, dom.mesh.elements[lo:lo + dom.num_owned])
        dt = stable_dt(own_mesh, _cg(own_mesh), args.order)  # identical on every rank (congruent slabs)
        u0_host = CavityMode(1, 1, 1, extent).evaluate(dom.owned_nodes(), 0.0)
    u = op.to_padded(u0_host)
    setup_s = time.perf_counter() - t_setup
    k = op.num_elements
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def advance(x, n):
        if world == 1:
            return op.advance(x, dt, n, use_graph=False)
        return runner.advance(x, dt, n)

    # ---- device-resident throughput (value) ----
    with ClockSampler(local) as clocks:
        advance(u, args.warmup)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks.mark_start()
        start.record(stream)
        advance(u, args.steps)
        stop.record(stream)
        torch.cuda.synchronize()
        clocks.mark_stop()
        time.sleep(0.15)  # let the sample covering the end of the timed region arrive
    barrier()
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    energy = runner.field_energy(u)
    if not math.isfinite(energy):
        raise RuntimeError("non-finite energy after the timed steps")

    launches = 5 * args.steps if world == 1 else args.steps * 5 * (
        1 + len(runner.stage_ranges()[1]) + len(runner.domain.send) + len(runner.domain.recv))
    sec = ms / 1e3
    f_alg = flops_per_element_stage(args.order)
    b_alg = bytes_per_element_stage(args.order, word)
    gflops = world * f_alg * k * 5 * args.steps / sec / 1e9
    dof_rate = world * dofs(args.order, k) * args.steps / sec
    hbm_gbs = b_alg * k * 5 * args.steps / sec / 1e9  # per GPU
    launch_s = sec / launches
    peaks = _peaks()
    ncu = _ncu_summary()
    traffic = ncu.get("tc_stage_kernel" if op.path == "tensor" else "stage_kernel", {}).get("dram_bytes_per_launch")
    fp32_peak_tf = 148 * 128 * 2 * (peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12

    # ---- end-to-end through the public API with host buffers ----
    # Every e2e step uploads its own input (the natural state in the e2e dtype, pinned host memory),
    # packs it, runs one LSRK4 step, unpacks and downloads the new state and the energy scalar.  The
    # steps are independent and pipelined over three streams: uploads in order on an H2D stream,
    # pack/step/unpack on the compute stream, downloads in order on a D2H stream, with events
    # recycling `--e2e-slots` device input buffers, so both copy engines stream back to back (PCIe
    # is full duplex) while the GPU computes.  Every byte counted below crosses PCIe inside the
    # timed region.
    e2e_steps = max(1, args.steps if args.e2e_steps is None else min(args.steps, args.e2e_steps))
    # natural host state in the e2e dtype (default: the compute dtype -- an fp32 user keeps fp32 host
    # buffers; --e2e-dtype f64 keeps the reference's float64 and doubles the PCIe bytes)
    e2e_dtype = {"f32": torch.float32, "f64": torch.float64}[args.e2e_dtype or args.dtype]
    host_in = torch.from_numpy(np.ascontiguousarray(u0_host)).to(e2e_dtype).pin_memory()
    nslots = max(2, args.e2e_slots)
    host_out = [torch.empty_like(host_in).pin_memory() for _ in range(nslots)]
    e_host = [torch.empty(1, dtype=torch.float64).pin_memory() for _ in range(nslots)]
    h2d = host_in.numel() * host_in.element_size()
    d2h = host_out[0].numel() * host_out[0].element_size() + 8
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    dev_in = [torch.empty(host_in.shape, dtype=e2e_dtype, device=dev) for _ in range(nslots)]
    ue = op.empty_state()  # one compute stream: the state buffer is reused in stream order
    in_ready = [torch.cuda.Event() for _ in range(nslots)]   # H2D into dev_in[j] done
    in_free = [torch.cuda.Event() for _ in range(nslots)]    # dev_in[j] packed (reusable)
    out_ready = [torch.cuda.Event() for _ in range(nslots)]  # slot j's result unpacked
    out_free = [torch.cuda.Event() for _ in range(nslots)]   # slot j's result downloaded
    used = [False] * nslots

    def e2e_step(i):
        j = i % nslots
        with torch.cuda.stream(h2d_s):
            if used[j]:
                h2d_s.wait_event(in_free[j])
            dev_in[j].copy_(host_in, non_blocking=True)                     # H2D
            in_ready[j].record(h2d_s)
        with torch.cuda.stream(stream):
            stream.wait_event(in_ready[j])
            op.to_padded(dev_in[j], out=ue)                                 # pack (natural -> padded)
            in_free[j].record(stream)
            advance(ue, 1)                                                  # 5 fused stage launches
            if used[j]:
                stream.wait_event(out_free[j])  # bounds the results in flight to nslots
            nat = op.from_padded(ue, e2e_dtype)                             # unpack
            energy_dev = op.mass_norm(ue, 1.0, 1.0)                         # per-step energy scalar
            nat.record_stream(d2h_s)
            energy_dev.record_stream(d2h_s)
            out_ready[j].record(stream)
        with torch.cuda.stream(d2h_s):
            d2h_s.wait_event(out_ready[j])
            host_out[j].copy_(nat, non_blocking=True)                       # D2H of the new state
            e_host[j].copy_(energy_dev, non_blocking=True)
            out_free[j].record(d2h_s)
        used[j] = True

    for j in range(nslots):  # warm-up (allocations, first launches)
        e2e_step(j)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e_start, e_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    h2d_s.wait_stream(stream)
    d2h_s.wait_stream(stream)
    for i in range(e2e_steps):
        e2e_step(i)
    stream.wait_stream(h2d_s)
    stream.wait_stream(d2h_s)
    e_stop.record(stream)
    torch.cuda.synchronize()
    barrier()
    e_ms = e_start.elapsed_time(e_stop)
    if world > 1:
        t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e_gflops = world * f_alg * k * 5 * e2e_steps / (e_ms / 1e3) / 1e9

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_rate(args.order, CPU_SAMPLE_CELLS, args.cpu_steps)
        cpu = {"value": r["gflops"], "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"oracle port of the reference path, box {CPU_SAMPLE_CELLS} -> {r['elements']} tets, "
                         f"N={args.order}, {args.cpu_steps} LSRK4 steps, {r['seconds']:.1f} s single-threaded; "
                         f"{r['dof_updates_per_s']:.3g} DOF-updates/s"}
    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": gflops, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if word == 8 else "f32", "data": "synthetic",
        "dof_updates_per_s": dof_rate, "hbm_gbs_algorithmic": hbm_gbs,
        "config": {"workload": f"C3 Maxwell PEC cavity N={args.order}, box {cells} -> {k} tets per GPU, "
                               "TM(1,1,1) cavity mode, dt=stable_dt(cfl=1)",
                   "order": args.order, "elements_per_gpu": k, "dofs_per_gpu": dofs(args.order, k),
                   "parallelism": f"x-slab element partition over {world} GPUs, NCCL face-trace halo "
                                  "overlapped with the interior stage kernel" if world > 1 else "single",
                   "global_elements": k * world,
                   "l2": "no flush: state+residual registers (%.2f GB) >> 126 MB L2" % (
                       2 * 6 * k * op.np_stride * word / 1e9),
                   "element_order": (args.element_order if args.element_order != "auto" else "columns")
                   if getattr(op, "_order", None) is not None else "natural",
                   "face_slots": "bank-spread" if getattr(op, "_slot_inv", None) is not None else "natural",
                   "setup_s": round(setup_s, 2), "flops_per_element_stage": f_alg,
                   "bytes_per_element_stage": b_alg},
        "roofline": {"bound": "hbm", "achieved": b_alg * k / launch_s / 1e9, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": b_alg * k / launch_s / 1e9 / peaks["hbm_gbs"],
                     "traffic": traffic,
                     "kernel": (f"dgm::tc_stage_kernel<{args.order},1>" if op.path == "tensor" else
                                f"dgm::stage_kernel<{args.order},{'float' if word == 4 else 'double'},1>"),
                     "path": op.path,
                     "launch_us": launch_s * 1e6,
                     "peak_source": peaks["source"],
                     "fp32_simt_frac": f_alg * k / launch_s / 1e12 / fp32_peak_tf,
                     "fp32_simt_peak_tflops": fp32_peak_tf},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_gflops, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "ms_per_step": e_ms / e2e_steps,
                "slots": nslots,
                "host_dtype": str(e2e_dtype).replace("torch.", ""),
                "path": "per step: pinned natural state H2D -> op.to_padded -> op.advance(1 LSRK4 step) -> "
                        "op.from_padded -> pinned host D2H, + energy scalar D2H; pipelined over an H2D, a "
                        "compute and a D2H stream with %d input slots" % nslots},
        "gpu_launches": launches,
        "clocks": clk,
        "energy_after": energy,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--order", type=int, default=ORDER)
    ap.add_argument("--cells", type=int, nargs=3, default=list(CELLS))
    ap.add_argument("--dtype", choices=("f32", "f64"), default="f32")
    ap.add_argument("--e2e-steps", type=int, default=None, help="e2e steps (default: --steps)")
    ap.add_argument("--e2e-slots", type=int, default=4,
                    help="device input buffers of the e2e pipeline (H2D runs up to this many steps ahead)")
    ap.add_argument("--element-order", choices=("auto", "natural", "morton", "columns"), default="auto",
                    help="internal element numbering (ordering.py); auto = Morton where it pays")
    ap.add_argument("--face-slots", choices=("auto", "natural"), default="auto",
                    help="node order inside each face (ordering.face_slot_order); auto = bank-spread on the tensor path")
    ap.add_argument("--e2e-dtype", choices=("f32", "f64"), default=None,
                    help="natural host-state dtype of the e2e leg (default: the compute dtype)")
    ap.add_argument("--cpu-steps", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--path", choices=("auto", "tensor", "simt"), default="auto",
                    help="stage kernel: tcgen05 3xTF32 (tensor, N<=4 fp32) or CUDA cores (simt)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
