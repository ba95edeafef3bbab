"""Benchmark of the B200 nodal-DG Maxwell operator (one JSON line on rank 0).

Workload (BASELINE.json configs[2], the metric's N=4 single-GPU config): PEC
cubic cavity, box (55,55,55) -> 998,250 tets, order N=4, fp32, TM (1,1,1)
cavity-mode initial state, dt = stable_dt(cfl=1).  A *step* is one LSRK4
step = 5 launches of the fused stage kernel over all elements.  The state
register (0.86 GB) and residual are far larger than the 126 MB L2, so no
explicit flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 runs under torchrun, one rank per GPU (NCCL); see DESIGN.md.
--impl reference times the reference itself (simtdg's build_reference_operator
.rhs inside its rk4_step, installed into baseline/_ref by
scripts/install_reference.sh; the oracle port if absent) on the host cores.

The N=1 line also carries the other BASELINE configs (C1 through the CUDA-graph
path, a C2 order subset, C3 fp64, C5 N=6) under "configs", each with its own
clocks and a max(B_alg/BW, F_alg/P) roofline; --extras selects them.
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
N_FIELDS_E2E = 6  # field slabs (E_x .. H_z) of the natural state, each copied in --e2e-chunks pieces
ORDER = 4
CELLS = (55, 55, 55)


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
        self.windows = {}  # name -> [t0, t1] of an extra config's timed region

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

    def mark_start(self, name: str | None = None):
        if name is None:
            self.t0 = time.time()
        else:
            self.windows[name] = [time.time(), None]

    def mark_stop(self, name: str | None = None):
        t = time.time() + 0.1  # the line reporting the last timed interval arrives a period later
        if name is None:
            self.t1 = t
        else:
            self.windows[name][1] = t

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=5)

    def summary(self, name: str | None = None) -> dict:
        t0, t1 = (self.t0, self.t1) if name is None else self.windows.get(name, (None, None))
        lines = [l for t, l in self.samples if t0 is not None and t0 <= t <= (t1 or t)]
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


# ----------------------------------------------------------------------------------------------
# CPU reference: the genuine simtdg (baseline/_ref, installed by scripts/install_reference.sh) when
# present, else the oracle port.  One single-threaded process per host core, each integrating its
# own x-slab of the C2 box (20^3 cells, 48,000 tets in total) with the reference's own
# build_reference_operator + rk4_step (numpy einsum is single-threaded, so processes are how the
# reference uses all host cores); rate = all workers' work / the slowest worker's time.
# ----------------------------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
CPU_SAMPLE_BOX = (20, 20, 20)
CPU_MAX_ELEMENTS_PER_WORKER = 7200  # ~2.5 s per N=4 step per worker: the whole run stays within minutes


def _host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _ref_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "simtdg"))


def _cpu_worker(kind, order, cx, x0, steps, warmup, barrier, queue):
    """One reference process: slab [x0, x0 + cx) x 20 x 20 cells of the unit C2 box."""
    import numpy as np

    if kind == "reference":
        sys.path.insert(0, REF_DIR)
        from simtdg.kernels.assemble import rk4_step
        from simtdg.kernels.oracle import build_reference_operator as build
        from simtdg.maxwell import CavityMode, stable_dt
        from simtdg.mesh import generate_box_mesh
        from simtdg.refelem import build_reference_element
    else:
        from oracle import build_oracle_operator as build
        from oracle import rk4_step
        from paper_0901_1024_b200 import CavityMode, build_reference_element, generate_box_mesh, stable_dt
    nx = CPU_SAMPLE_BOX[0]
    mesh = generate_box_mesh((cx / nx, 1.0, 1.0), (cx, CPU_SAMPLE_BOX[1], CPU_SAMPLE_BOX[2]))
    mesh.vertices[:, 0] += x0 / nx
    elem = build_reference_element(order)
    op = build(mesh, elem)
    u = CavityMode(1, 1, 1, extent=(1.0, 1.0, 1.0)).evaluate(op.nodes, 0.0)
    dt = stable_dt(mesh, op.geometry, order)
    for _ in range(warmup):
        u = rk4_step(u, 0.0, dt, lambda t, y: op.rhs(y))
    barrier.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        u = rk4_step(u, 0.0, dt, lambda t, y: op.rhs(y))
    sec = time.perf_counter() - t0
    queue.put((int(mesh.elements.shape[0]), sec, bool(np.isfinite(u).all())))


def cpu_reference_rate(order: int, steps: int, warmup: int = 0, workers: int | None = None) -> dict:
    """Time the reference path on the host cores (see the block comment above)."""
    import multiprocessing as mp

    from paper_0901_1024_b200.perfmodel import flops_per_element_stage
    from paper_0901_1024_b200.refelem import simplex_node_count

    kind = "reference" if _ref_available() else "port"
    cores = _host_cores()
    p = max(1, min(workers or cores, CPU_SAMPLE_BOX[0]))
    nx, ny, nz = CPU_SAMPLE_BOX
    per_x = 6 * ny * nz
    # slabs of >= 1 x-cell, at most CPU_MAX_ELEMENTS_PER_WORKER tets each (smaller sample on few cores)
    cx_max = max(1, CPU_MAX_ELEMENTS_PER_WORKER // per_x)
    total_x = min(nx, p * cx_max)
    base, extra = divmod(total_x, p)
    slabs, x0 = [], 0
    for i in range(p):
        cx = base + (1 if i < extra else 0)
        if cx:
            slabs.append((cx, x0))
            x0 += cx
    env_keep = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env_keep:
        os.environ[k] = "1"  # one core per worker (inherited by the spawned processes)
    ctx = mp.get_context("spawn")
    barrier, queue = ctx.Barrier(len(slabs)), ctx.Queue()
    procs = [ctx.Process(target=_cpu_worker, args=(kind, order, cx, x0, steps, warmup, barrier, queue))
             for cx, x0 in slabs]
    try:
        for pr in procs:
            pr.start()
        res = [queue.get(timeout=1800) for _ in procs]
        for pr in procs:
            pr.join()
    finally:
        for k, v in env_keep.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    if not all(r[2] for r in res):
        raise RuntimeError("non-finite state in the CPU reference run")
    k = sum(r[0] for r in res)
    sec = max(r[1] for r in res)
    n_p = simplex_node_count(order)[0]
    flops = flops_per_element_stage(order) * k * 5 * steps
    path = ("genuine simtdg 0.1.0 (baseline/_ref) build_reference_operator().rhs inside simtdg rk4_step"
            if kind == "reference" else "oracle port (oracle/dg_oracle.py) of simtdg rhs + rk4_step")
    sample = (f"{len(slabs)} single-threaded processes x one x-slab each of the C2 box {CPU_SAMPLE_BOX} "
              f"({k} tets in total, N={order}), {steps} LSRK4 steps after {warmup} warm-up; {path}; "
              f"rate per DOF is nearly K-independent, so it stands for the named config")
    return {"gflops": flops / sec / 1e9, "dof_updates_per_s": 6 * n_p * k * steps / sec, "seconds": sec,
            "elements": k, "steps": steps, "kind": kind, "cores": len(slabs), "host_cores": cores,
            "sample": sample}


def run_reference(args) -> None:
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    r = cpu_reference_rate(args.order, args.steps, args.warmup)
    line = {
        "metric": METRIC, "value": r["gflops"], "unit": UNIT, "impl": "reference", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "dof_updates_per_s": r["dof_updates_per_s"],
        "config": {"workload": f"C3 Maxwell PEC cavity N={args.order}, box {tuple(args.cells)} (per-DOF rate "
                               f"on a bounded sample, see cpu_baseline.sample)", "order": args.order,
                   "sample_elements": r["elements"], "host_cores": r["host_cores"]},
        "cpu_baseline": {"value": r["gflops"], "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "host_cores": r["host_cores"], "sample": r["sample"]},
        "e2e": {"value": r["gflops"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
# Roofline: T_roof = max(B_alg / BW, F_alg / P) per element-stage; P is the peak of
# the pipe the kernel computes on: the measured kind::tf32 MMA rate / 3 for the 3xTF32 tensor path,
# FP32 or FP64 SIMT (148 SMs x 128 / 64 lanes x 2 flop x clock) otherwise.
# ----------------------------------------------------------------------------------------------
def measure_tf32_tflops(dev, sm_mhz: float) -> dict | None:
    """kind::tf32 MMA throughput of one SM (probe library, M=128 N=48 K=8 TS bursts) x SMs x clock."""
    import ctypes

    import torch

    path = os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so")
    try:
        lib = ctypes.CDLL(path)
    except OSError:
        return None
    lib.dgm_probe_mma_rate.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
    out = torch.zeros(2, dtype=torch.int64, device=dev)
    best = None
    with torch.cuda.device(dev):
        for _ in range(3):
            if lib.dgm_probe_mma_rate(48, 960, 1, 0, out.data_ptr()) != 0:
                return None
            torch.cuda.synchronize(dev)
            clk = out[1].item() / 960.0
            best = clk if best is None else min(best, clk)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    flop_clk = 128 * 48 * 8 * 2 / best
    return {"tflops": flop_clk * sms * sm_mhz * 1e6 / 1e12, "clk_per_mma": best, "sms": sms,
            "source": "probe: tcgen05.mma kind::tf32 M=128 N=48 K=8 (A in TMEM) bursts, measured in this run"}


def measure_fp64_tflops(dev) -> dict | None:
    """FP64 throughput of this GPU, measured in this run: DMMA (mma.sync m8n8k4 f64, the tensor pipe the
    fp64 stage kernel's volume and LIFT products run on for N <= 6) and DFMA (the CUDA cores)."""
    import ctypes

    import torch

    try:
        lib = ctypes.CDLL(os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so"))
    except OSError:
        return None
    lib.dgm_probe_fp64_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    out = {}
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        for name, tensor, flop_iter in (("dmma", 1, 8 * 8 * 512), ("dfma", 0, 256 * 8 * 2)):
            blocks, iters = 8 * sms, 4096
            best = None
            for _ in range(3):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                if lib.dgm_probe_fp64_rate(tensor, blocks, iters, sink.data_ptr(), stream.cuda_stream) != 0:
                    return None
                e.record(stream)
                torch.cuda.synchronize(dev)
                ms = s.elapsed_time(e)
                best = ms if best is None else min(best, ms)
            out[name + "_tflops"] = blocks * iters * flop_iter / (best / 1e3) / 1e12
    out["source"] = "probe kernels (8 blocks/SM x 8 warps, 8 independent chains), measured in this run"
    return out


def roofline(order, word, path, k, launch_s, peaks, pipes, kernel, traffic):
    from paper_0901_1024_b200.perfmodel import bytes_per_element_stage, flops_per_element_stage

    b = bytes_per_element_stage(order, word) * k
    f = flops_per_element_stage(order) * k
    bw = peaks["hbm_gbs"] * 1e9
    if path in ("tensor", "tensor2") and pipes.get("tf32"):
        p, pipe = pipes["tf32"]["tflops"] * 1e12 / 3.0, "tensor"
        psrc = "3xTF32: measured kind::tf32 rate / 3 (" + pipes["tf32"]["source"] + ")"
    elif word == 8 and order <= 6 and pipes.get("fp64"):
        # fp64 N <= 6: volume + LIFT on DMMA, the rest on the CUDA cores; the faster measured pipe bounds it
        f64 = pipes["fp64"]
        p = max(f64["dmma_tflops"], f64["dfma_tflops"]) * 1e12
        pipe, psrc = "fp64", ("FP64 (DMMA volume/LIFT): max of the measured DMMA %.1f and DFMA %.1f TFLOP/s (%s)"
                              % (f64["dmma_tflops"], f64["dfma_tflops"], f64["source"]))
    elif word == 8:
        p, pipe, psrc = pipes["fp64_tflops"] * 1e12, "fp64", "FP64 SIMT: SMs x 64 x 2 x max SM clock"
    else:
        p, pipe, psrc = pipes["fp32_tflops"] * 1e12, "fp32", "FP32 SIMT: SMs x 128 x 2 x max SM clock"
    t_mem, t_cmp = b / bw, f / p
    hbm = t_mem >= t_cmp
    return {"bound": "hbm" if hbm else pipe,
            "achieved": (b if hbm else f) / launch_s / (1e9 if hbm else 1e12),
            "peak": peaks["hbm_gbs"] if hbm else p / 1e12,
            "unit": "GB/s" if hbm else "TFLOP/s",
            "frac": max(t_mem, t_cmp) / launch_s,
            "traffic": traffic["bytes_per_launch"] if traffic else None,  # ncu DRAM bytes per launch
            "traffic_source": traffic,
            "kernel": kernel, "path": path, "launch_us": launch_s * 1e6,
            "t_roof_us": max(t_mem, t_cmp) * 1e6, "hbm_term_us": t_mem * 1e6, "compute_term_us": t_cmp * 1e6,
            "hbm_frac": t_mem / launch_s, "compute_frac": t_cmp / launch_s,
            "compute_peak_tflops": p / 1e12, "compute_peak_source": psrc,
            "peak_source": peaks["source"] if hbm else psrc}


def _kernel_name(order, word, path):
    if path == "tensor2":
        return f"dgm::tc2_stage_kernel<{order},1>"
    if path == "tensor":
        return f"dgm::tc_stage_kernel<{order},1>"
    return f"dgm::stage_kernel<{order},{'float' if word == 4 else 'double'},1>"


def _traffic(ncu: dict, order: int, word: int, path: str, elements: int):
    """ncu DRAM bytes per launch of this (kernel, order, dtype, mesh size), or None if not captured."""
    fam = {"tensor": "tc_stage_kernel", "tensor2": "tc2_stage_kernel"}.get(path, "stage_kernel")
    key = f"{fam}<{order}>/{'f32' if word == 4 else 'f64'}@{elements}"
    ent = ncu.get("kernels", {}).get(key)
    return {"bytes_per_launch": ent["dram_bytes_per_launch"], "key": key, "source": ent.get("source")} if ent else None


# Extra config rows timed in the same N=1 run (BASELINE.json configs).
EXTRAS = {
    "C1": dict(order=3, cells=(6, 6, 7), dtype="f32", steps=100, warmup=10, graph=True,
               what="C1 PEC cavity N=3, 1,512 tets, 100 LSRK4 steps through the CUDA-graph path (op.advance)"),
    **{"C2_N%d" % n: dict(order=n, cells=(20, 20, 20), dtype="f32", steps=20 if n < 9 else 10, warmup=3,
                          graph=False, what="C2 order sweep, 48,000 tets, N=%d" % n) for n in range(1, 10)},
    "C3_f64": dict(order=4, cells=(55, 55, 55), dtype="f64", steps=10, warmup=3, graph=False,
                   what="C3 N=4, 998,250 tets, fp64 variant (the reference's precision)"),
    "C5": dict(order=6, cells=(70, 70, 70), dtype="f32", steps=10, warmup=3, graph=False,
               what="C5 N=6, 2,058,000 tets per GPU (N=1 point of the weak-scaling series), 3xTF32 tensor path"),
    "C4": dict(order=4, cells=(110, 110, 110), dtype="f32", steps=5, warmup=3, graph=False,
               what="C4 N=4, 7,986,000 tets on one GPU (N=1 point of the strong-scaling series)"),
}
DEFAULT_EXTRAS = ("C1",) + tuple("C2_N%d" % n for n in range(1, 10)) + ("C3_f64", "C5", "C4")


def run_extra(name, spec, dev, clocks, peaks, pipes, ncu) -> dict:
    """Build and time one extra config (device-resident state, CUDA events on the launching stream)."""
    import torch

    from paper_0901_1024_b200 import (CavityMode, build_b200_operator, build_reference_element,
                                      generate_box_mesh, map_nodes, stable_dt)
    from paper_0901_1024_b200.perfmodel import dofs, flops_per_element_stage

    t0 = time.perf_counter()
    dtype = torch.float64 if spec["dtype"] == "f64" else torch.float32
    word = 8 if dtype == torch.float64 else 4
    mesh = generate_box_mesh((1.0, 1.0, 1.0), spec["cells"])
    elem = build_reference_element(spec["order"])
    op = build_b200_operator(mesh, elem, dtype=dtype, device=dev)
    dt = stable_dt(mesh, op.geometry, spec["order"])
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream(dev)
    op.advance(u, dt, spec["warmup"], use_graph=spec["graph"])
    torch.cuda.synchronize(dev)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark_start(name)
    start.record(stream)
    op.advance(u, dt, spec["steps"], use_graph=spec["graph"])
    stop.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark_stop(name)
    ms = start.elapsed_time(stop)
    energy = op.field_energy(u)
    if not math.isfinite(energy):
        raise RuntimeError(f"{name}: non-finite energy")
    k, order, steps = op.num_elements, spec["order"], spec["steps"]
    sec = ms / 1e3
    launch_s = sec / (5 * steps)
    out = {"workload": spec["what"], "order": order, "elements": k, "dtype": spec["dtype"], "path": op.path,
           "steps": steps, "warmup": spec["warmup"], "cuda_graph": spec["graph"], "ms_per_step": ms / steps,
           "value": flops_per_element_stage(order) * k * 5 * steps / sec / 1e9, "unit": UNIT,
           "dof_updates_per_s": dofs(order, k) * steps / sec, "setup_s": round(setup_s, 2),
           "roofline": roofline(order, word, op.path, k, launch_s, peaks, pipes, _kernel_name(order, word, op.path),
                                _traffic(ncu, order, word, op.path, k)),
           "energy_after": energy}
    del op, u
    torch.cuda.empty_cache()
    time.sleep(0.15)
    out["clocks"] = clocks.summary(name)
    return out


def run_b200(args) -> None:
    import numpy as np
    import torch

    from paper_0901_1024_b200 import (CavityMode, build_b200_operator, build_reference_element, compute_geometry,
                                      generate_box_mesh, map_nodes, stable_dt)
    from paper_0901_1024_b200.perfmodel import bytes_per_element_stage, dofs, flops_per_element_stage
    from paper_0901_1024_b200.hoststep import HostStepper

    world, rank, local = _dist_env()
    # DGM_BENCH_ONE_GPU=1 (testing only): every rank on device 0, to exercise the N > 1 path on a
    # single-GPU box (NCCL permitting); never set for a reported number
    gpu = 0 if os.environ.get("DGM_BENCH_ONE_GPU") == "1" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        import torch.distributed as dist

        if os.environ.get("DGM_BENCH_ONE_GPU") == "1":  # testing the N > 1 path on one GPU: gloo
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    dtype = torch.float64 if args.dtype == "f64" else torch.float32
    word = 8 if dtype == torch.float64 else 4
    cells = tuple(args.cells)
    strong = args.scaling == "strong" and world > 1
    t_setup = time.perf_counter()
    elem = build_reference_element(args.order)
    if world == 1:
        mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
        op = build_b200_operator(mesh, elem, dtype=dtype, device=dev, path=args.path,
                                 reorder={"auto": None, "natural": False, "morton": "morton",
                                          "columns": True, "greedy": "greedy"}[args.element_order],
                                 face_slots=None if args.face_slots == "auto" else False)
        dt = stable_dt(mesh, op.geometry, args.order)
        extent = (1.0, 1.0, 1.0)
        u0_host = CavityMode(1, 1, 1, extent).evaluate(map_nodes(mesh, elem), 0.0)
        runner = op
    else:
        from paper_0901_1024_b200.dist import DistributedMaxwellOperator, build_box_domain
        from paper_0901_1024_b200.mesh import Mesh, compute_geometry as _cg

        if strong:
            # strong scaling: the (cells) box split into world x-slabs (C4: 110^3 over 1/2/4/8 GPUs)
            extent, gcells = (1.0, 1.0, 1.0), cells
        else:
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
        dt_local = stable_dt(own_mesh, _cg(own_mesh), args.order)
        t = torch.tensor([dt_local], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)  # global stable dt
        dt = float(t.item())
        u0_host = CavityMode(1, 1, 1, extent).evaluate(dom.owned_nodes(), 0.0)
    u = op.to_padded(u0_host)
    setup_s = time.perf_counter() - t_setup
    k = op.num_elements
    path = op.path
    launches = 5 * args.steps if world == 1 else args.steps * 5 * (
        1 + len(runner.stage_ranges()[1]) + len(runner.domain.send) + len(runner.domain.recv))
    k_total = k
    if world > 1:
        t = torch.tensor([k], device=dev, dtype=torch.int64)
        torch.distributed.all_reduce(t)
        k_total = int(t.item())
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def advance(x, n):
        if world == 1:
            return op.advance(x, dt, n, use_graph=False)
        return runner.advance(x, dt, n)

    def max_over_ranks(ms):
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    peaks = _peaks()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    pipes = {"fp32_tflops": sms * 128 * 2 * sm_max * 1e6 / 1e12, "fp64_tflops": sms * 64 * 2 * sm_max * 1e6 / 1e12,
             "tf32": measure_tf32_tflops(dev, sm_max), "fp64": measure_fp64_tflops(dev)}
    ncu = _ncu_summary()

    with ClockSampler(gpu) as clocks:
        # ---- device-resident throughput (value) ----
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
        barrier()
        torch.cuda.synchronize()
        ms = max_over_ranks(start.elapsed_time(stop))
        energy = runner.field_energy(u)
        if not math.isfinite(energy):
            raise RuntimeError("non-finite energy after the timed steps")

        # ---- end to end through the public API with host buffers (a dependent chain) ----
        # The reference user's state lives on the host in float64 (natural (6, K, Np) layout).  Every
        # e2e step is one HostStepper.step call (paper_0901_1024_b200/hoststep.py): upload the current
        # host state (pinned), pack, one LSRK4 step, unpack, download the new state into the same host
        # buffer -- the next step's input -- plus the energy scalar.  The upload of piece p for step i+1
        # waits for the download of piece p from step i and the pack waits for every upload, so every
        # step computes on the previous step's downloaded output; what overlaps is the download of step
        # i with the upload of step i+1 (PCIe is full duplex).  --e2e-serial: one copy per direction.
        e2e_steps = max(1, args.steps if args.e2e_steps is None else min(args.steps, args.e2e_steps))
        e2e_dtype = {"f32": torch.float32, "f64": torch.float64}[args.e2e_dtype]
        host = torch.from_numpy(np.ascontiguousarray(u0_host)).to(e2e_dtype).pin_memory()
        e_host = torch.zeros(1, dtype=torch.float64).pin_memory()
        h2d = host.numel() * host.element_size()
        d2h = h2d + 8
        stepper = HostStepper(op, advance=lambda x, dt_, n: advance(x, n), chunks=args.e2e_chunks,
                              serial=args.e2e_serial)
        stepper.step(host, dt, 1, energy_out=e_host)  # warm-up (allocations, first launches)
        stepper.join()
        torch.cuda.synchronize()
        host.copy_(torch.from_numpy(np.ascontiguousarray(u0_host)).to(e2e_dtype))
        barrier()
        torch.cuda.synchronize()
        e_start, e_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        for _ in range(e2e_steps):  # one public-API call per step, as a user's loop would make them
            stepper.step(host, dt, 1, energy_out=e_host)
        stepper.join()  # the last download is inside the timed region
        e_stop.record(stream)
        torch.cuda.synchronize()
        barrier()
        e_ms = max_over_ranks(e_start.elapsed_time(e_stop))
        if not math.isfinite(float(e_host.item())):
            raise RuntimeError("non-finite e2e energy")
        pieces = len(stepper._buffers(e2e_dtype)["pieces"])
        del stepper

        # ---- the RHS-level drop-in, as the reference's own loop calls it (N=1 only) ----
        # rk4_step(state, t, dt, lambda t, y: op.rhs(y)) on a float64 numpy state: every RHS call
        # round-trips the state through pageable host memory and the LSRK arithmetic runs in numpy
        # on the host (stepper.py:49-70 = assemble.py:105-114).  Host wall clock (the host work is the
        # point), one warm-up RHS call, then `--dropin-steps` dependent steps.
        dropin = None
        if world == 1 and args.dropin_steps > 0:
            from paper_0901_1024_b200.stepper import rk4_step as host_rk4_step

            y = np.array(u0_host, dtype=np.float64)
            op.rhs(y)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.dropin_steps):
                y = host_rk4_step(y, 0.0, dt, lambda t, v: op.rhs(v))
            torch.cuda.synchronize()
            d_s = time.perf_counter() - t0
            if not np.isfinite(y).all():
                raise RuntimeError("non-finite drop-in state")
            dropin = {"value": flops_per_element_stage(args.order) * k * 5 * args.dropin_steps / d_s / 1e9,
                      "unit": UNIT, "steps": args.dropin_steps, "ms_per_step": d_s * 1e3 / args.dropin_steps,
                      "h2d_bytes_per_step": 5 * y.nbytes, "d2h_bytes_per_step": 5 * y.nbytes,
                      "timing": "host wall clock",
                      "path": "reference call pattern: rk4_step(numpy float64 state, t, dt, lambda t, y: op.rhs(y)) "
                              "-- per RHS: pageable H2D, pack, dgm_rhs, unpack, D2H; LSRK arithmetic in numpy"}
            del y

        # ---- the other BASELINE configs on this GPU (N=1 only) ----
        extras = {}
        if world == 1 and args.extras != "none":
            del u
            runner = op = None
            torch.cuda.empty_cache()
            names = DEFAULT_EXTRAS if args.extras == "default" else (
                tuple(EXTRAS) if args.extras == "all" else tuple(args.extras.split(",")))
            for name in names:
                extras[name] = run_extra(name, EXTRAS[name], dev, clocks, peaks, pipes, ncu)
        time.sleep(0.15)  # let the sample covering the end of the last timed region arrive

    sec = ms / 1e3
    f_alg = flops_per_element_stage(args.order)
    b_alg = bytes_per_element_stage(args.order, word)
    gflops = f_alg * k_total * 5 * args.steps / sec / 1e9
    dof_rate = dofs(args.order, k_total) * args.steps / sec
    hbm_gbs = b_alg * k * 5 * args.steps / sec / 1e9  # per GPU
    launch_s = sec / (5 * args.steps)
    e2e_gflops = f_alg * k_total * 5 * e2e_steps / (e_ms / 1e3) / 1e9

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_rate(args.order, args.cpu_steps, 1)
        cpu = {"value": r["gflops"], "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
               "host_cores": r["host_cores"], "sample": r["sample"],
               "dof_updates_per_s": r["dof_updates_per_s"]}
    clk = clocks.summary()
    if world == 1:
        parallelism = "single"
    elif strong:
        parallelism = (f"strong scaling: the {cells} box split into {world} x-slabs, NCCL face-trace halo "
                       "overlapped with the interior stage kernel")
    else:
        parallelism = (f"weak scaling: {world} x-slabs of {cells} cells each, NCCL face-trace halo "
                       "overlapped with the interior stage kernel")
    line = {
        "metric": METRIC, "value": gflops, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f64" if word == 8 else "f32", "data": "synthetic",
        "dof_updates_per_s": dof_rate, "hbm_gbs_algorithmic": hbm_gbs,
        "config": {"workload": (f"C4 Maxwell PEC cavity N={args.order}, box {cells} -> {k_total} tets over "
                                f"{world} GPUs" if strong else
                                f"C3 Maxwell PEC cavity N={args.order}, box {cells} -> {k} tets per GPU") +
                               ", TM(1,1,1) cavity mode, dt=stable_dt(cfl=1)",
                   "order": args.order, "elements_per_gpu": k, "dofs_per_gpu": dofs(args.order, k),
                   "parallelism": parallelism, "global_elements": k_total,
                   "l2": "no flush: state+residual registers (%.2f GB) >> 126 MB L2" % (
                       2 * 6 * k * _np_stride(args.order, word) * word / 1e9),
                   "setup_s": round(setup_s, 2), "flops_per_element_stage": f_alg,
                   "bytes_per_element_stage": b_alg},
        "roofline": roofline(args.order, word, path, k, launch_s, peaks, pipes,
                             _kernel_name(args.order, word, path), _traffic(ncu, args.order, word, path, k)),
        "cpu_baseline": cpu,
        "dropin_rhs": dropin,
        "e2e": {"value": e2e_gflops, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "ms_per_step": e_ms / e2e_steps,
                "host_dtype": str(e2e_dtype).replace("torch.", ""),
                "overlap": "none (--e2e-serial)" if args.e2e_serial else (
                    "%d contiguous pieces: the upload of piece p for step i+1 waits for the download of "
                    "piece p from step i; the pack waits for every upload (download of step i overlaps "
                    "upload of step i+1, full-duplex PCIe)" % pieces),
                "path": "dependent chain through the public API, one HostStepper.step per step: pinned natural "
                        "host state H2D -> op.to_padded -> advance(1 LSRK4 step) -> op.from_padded -> D2H "
                        "into the same host buffer (the next step's input) + energy scalar D2H"},
        "gpu_launches": launches,
        "clocks": clk,
        "energy_after": energy,
        "pipes": {"fp32_simt_tflops": pipes["fp32_tflops"], "fp64_simt_tflops": pipes["fp64_tflops"],
                  "tf32_mma": pipes["tf32"], "fp64_measured": pipes["fp64"]},
    }
    if extras:
        line["configs"] = extras
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _np_stride(order: int, word: int) -> int:
    from paper_0901_1024_b200 import _capi

    return _capi.layout(order, _capi.DGM_F64 if word == 8 else _capi.DGM_F32).np_stride


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--order", type=int, default=ORDER)
    ap.add_argument("--cells", type=int, nargs=3, default=None,
                    help="box cells (default: C3 (55,55,55); with --scaling strong: C4 (110,110,110))")
    ap.add_argument("--dtype", choices=("f32", "f64"), default="f32")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="N>1: weak = --cells per GPU (C3/C5 style), strong = --cells split over the GPUs (C4)")
    ap.add_argument("--extras", default="default",
                    help="extra config rows at N=1: default (%s), all, none, or a comma list of %s"
                         % (",".join(DEFAULT_EXTRAS), ",".join(EXTRAS)))
    ap.add_argument("--e2e-steps", type=int, default=None, help="e2e steps (default: --steps)")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="e2e copy pieces per field slab")
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e copies as one H2D and one D2H per step, nothing overlapped")
    ap.add_argument("--dropin-steps", type=int, default=1,
                    help="steps of the RHS-level drop-in leg (reference call pattern, host numpy LSRK; 0: skip)")
    ap.add_argument("--element-order", choices=("auto", "natural", "morton", "columns", "greedy"), default="auto",
                    help="internal element numbering (ordering.py); auto = Morton where it pays")
    ap.add_argument("--face-slots", choices=("auto", "natural"), default="auto",
                    help="node order inside each face (ordering.face_slot_order); auto = bank-spread on the tensor path")
    ap.add_argument("--e2e-dtype", choices=("f32", "f64"), default="f64",
                    help="natural host-state dtype of the e2e leg (default: float64, the reference's)")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--path", choices=("auto", "tensor2", "tensor", "simt"), default="auto",
                    help="stage kernel: tcgen05 3xTF32 v2 (tensor2, N<=4 fp32) or v1 (tensor), or CUDA cores (simt)")
    args = ap.parse_args(argv)
    if args.cells is None:
        args.cells = [110, 110, 110] if args.scaling == "strong" else list(CELLS)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.extras not in ("default", "all", "none"):
        bad = [n for n in args.extras.split(",") if n not in EXTRAS]
        if bad:
            raise SystemExit(f"unknown --extras {bad}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
