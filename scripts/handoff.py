"""Producer/MMA hand-off primitive costs (probe library)."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so"))
lib.dgm_probe_handoff.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
reps = 400
for ctas in (1, 296):
    for mode in (0, 1):
        for pw in (4, 8):
            assert lib.dgm_probe_handoff(reps, mode, pw, ctas, out.data_ptr()) == 0
            torch.cuda.synchronize()
            print(f"ctas={ctas:3d} mode={mode} producer warps={pw}: {out[0].item() / reps:7.1f} cyc/iteration")
