"""tcgen05 kind::tf32 issue/completion rate (probe library)."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so"))
lib.dgm_probe_mma_rate.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for ts in (0, 1, 2):
    for n in (16, 48, 64, 128, 256):
        for nacc in (0, 1, 6):
            if (nacc != 1 and n > 64) or (ts == 2 and nacc == 6):
                continue
            reps = 1008 if nacc else 1008 // 48 * 48
            assert lib.dgm_probe_mma_rate(n, reps, ts, nacc, out.data_ptr()) == 0
            torch.cuda.synchronize()
            issue, done = out.tolist()
            print(f"{['SS-tf32', 'TS-tf32', 'SS-bf16'][ts]} N={n:3d} nacc={nacc}: issue {issue / reps:6.1f} cyc/MMA, "
                  f"complete {done / reps:6.1f} cyc/MMA  (ideal {128 * n / 256:5.1f})")
