"""Issue / round-trip cost of the stage kernel's per-K-step MMA burst in different shapes (probe library)."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so"))
lib.dgm_probe_mma_shape.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p]
names = ["3acc x 3pass pass-major, 1 commit", "3acc x 3pass pass-major, 2 commits", "3acc x 3pass acc-major",
         "9 independent accumulators", "6acc x 3pass (18 MMAs)", "2 K-steps (18 MMAs, 3acc) per burst"]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
reps = 300
for ctas in (148, 296):
    for v, name in enumerate(names):
        assert lib.dgm_probe_mma_shape(reps, v, ctas, out.data_ptr()) == 0
        torch.cuda.synchronize()
        tot, issue = out.tolist()
        print(f"ctas={ctas} {name:40s}: round trip {tot / reps:7.1f} cyc, issue {issue / reps:7.1f} cyc")
