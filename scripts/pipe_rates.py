"""Measured arithmetic pipe rates on this GPU (probe library): tcgen05 TF32, mma.sync TF32, DMMA, DFMA."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
out = {"tcgen05_tf32": bench.measure_tf32_tflops(dev, 1965.0), "fp64": bench.measure_fp64_tflops(dev)}
lib = ctypes.CDLL(os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so"))
lib.dgm_probe_tf32sync_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
sink = torch.zeros(1, device=dev)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
blocks, iters = 8 * sms, 4096
best = None
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    assert lib.dgm_probe_tf32sync_rate(blocks, iters, sink.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    best = ms if best is None else min(best, ms)
out["mma_sync_tf32_tflops"] = blocks * 8 * iters * 8 * 2048 / (best / 1e3) / 1e12
print(json.dumps(out, indent=1))
# DMMA and DFMA in one kernel (alternate warps): about the sum of the two rates if they are separate
# pipes, about either one if they share the FP64 datapath
lib.dgm_probe_fp64_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
sink64 = torch.zeros(1, dtype=torch.float64, device=dev)
best = None
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    assert lib.dgm_probe_fp64_rate(2, blocks, iters, sink64.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    best = ms if best is None else min(best, ms)
out["fp64_mixed_tflops"] = blocks * (4 * iters * 8 * 512 + 128 * iters * 8 * 2) / (best / 1e3) / 1e12
print(json.dumps({"fp64_mixed_tflops": out["fp64_mixed_tflops"]}))
