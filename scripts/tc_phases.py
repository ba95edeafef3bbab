"""Per-CTA phase durations of the tensor-core stage kernel (timing build libdgm_timing.so)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("DGM_LIB", os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_timing.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0901_1024_b200 import CavityMode, build_b200_operator, build_reference_element, generate_box_mesh, map_nodes  # noqa: E402
from paper_0901_1024_b200 import _capi  # noqa: E402

cells = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (30, 30, 30)
order = int(sys.argv[4]) if len(sys.argv) > 4 else 4
mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
elem = build_reference_element(order)
op = build_b200_operator(mesh, elem, path="tensor")
u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
op.advance(u, 1e-4, 2, use_graph=False)
bufs = op._buffers()
torch.cuda.synchronize()
op.lsrk_stage(u, bufs.alt, bufs.res, -0.4, 0.3, 1e-4)
torch.cuda.synchronize()
lib = _capi.load()
lib.dgm_phase_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
ntiles = min((mesh.num_elements + 63) // 64, 1 << 16)
buf = np.zeros((ntiles, 5), dtype=np.int64)
lib.dgm_phase_read(buf.ctypes.data, ntiles)
buf = buf[buf[:, 4] > 0]  # persistent kernel: one row per CTA (its last tile)
ntiles = len(buf)
d = np.diff(buf, axis=1)
names = ["start->rows landed", "rows->K-loop done", "K-loop->acc ready", "acc->epilogue done"]
print(f"{ntiles} CTAs, N={order}; cycles per CTA (mean / median / p90):")
for i, n in enumerate(names):
    print(f"  {n:22s} {d[:, i].mean():9.0f} {np.median(d[:, i]):9.0f} {np.percentile(d[:, i], 90):9.0f}")
tot = buf[:, 4] - buf[:, 0]
print(f"  {'total':22s} {tot.mean():9.0f} {np.median(tot):9.0f} {np.percentile(tot, 90):9.0f}")
