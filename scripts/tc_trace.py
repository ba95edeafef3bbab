"""Phase timeline of the tensor-core stage kernel (CTA 0), using the trace build libdgm_trace.so."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("DGM_LIB", os.path.join(ROOT, "paper_0901_1024_b200", "libdgm_trace.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0901_1024_b200 import (CavityMode, build_b200_operator, build_reference_element,  # noqa: E402
                                  generate_box_mesh, map_nodes)
from paper_0901_1024_b200 import _capi  # noqa: E402

cells = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (30, 30, 30)
order = int(sys.argv[4]) if len(sys.argv) > 4 else 4
mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
elem = build_reference_element(order)
op = build_b200_operator(mesh, elem, path="tensor")
u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
lib = _capi.load()
lib.dgm_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.dgm_hang_read.argtypes = [ctypes.c_void_p]
try:
    op.advance(u, 1e-4, 1, use_graph=False)
    op.lsrk_stage(u, op._buffers().alt, op._buffers().res, -0.4, 0.3, 1e-4)
    torch.cuda.synchronize()
except Exception as exc:  # noqa: BLE001
    print("kernel error:", exc)
hang = np.zeros(8, dtype=np.uint32)
lib.dgm_hang_read(hang.ctypes.data)
print("hang record (flag, block, thread, smem addr, parity):", hang[:5].tolist())
evs = []
for who in (0, 1):
    buf = np.zeros(2 * 4096, dtype=np.int64)
    n = lib.dgm_trace_read(buf.ctypes.data, who)
    evs.append(buf[: 2 * n].reshape(-1, 2))
ev = np.concatenate(evs)
ev = ev[np.argsort(ev[:, 1], kind="stable")]
t0 = ev[0, 1]
for tag, t in ev:
    print(f"{t - t0:9d}  {tag}")
