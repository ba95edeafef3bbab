"""Round-trip latency of MMA bursts (issue -> commit observed), stage-kernel pattern (probe library)."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_probe.so"))
lib.dgm_probe_mma_burst.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p]
out = torch.zeros(2, dtype=torch.int64, device="cuda")
reps = 200
for ctas in (1, 296):
    for n, nacc, passes in ((48, 3, 3), (48, 3, 1), (48, 1, 1), (48, 1, 9), (48, 4, 3), (16, 3, 3), (32, 3, 3), (64, 3, 3)):
        assert lib.dgm_probe_mma_burst(n, reps, nacc, passes, ctas, out.data_ptr()) == 0
        torch.cuda.synchronize()
        tot, issue = out.tolist()
        print(f"ctas={ctas:3d} N={n:3d} acc={nacc} passes={passes}: round trip {tot / reps:7.1f} cyc/burst "
              f"({tot / reps / (nacc * passes):6.1f}/MMA), issue {issue / reps:6.1f} cyc/burst")
