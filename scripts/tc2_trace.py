"""Phase timeline of the v2 stage kernel in CTA 0 (trace build libdgm_trace.so): producer tid 0 (P) and
the MMA-issuing epilogue warp (E), per tile: cycles since the first event."""
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

NAMES = {1: "P top", 2: "P tile landed", 3: "P stage_free", 4: "P split0", 5: "P split1", 6: "P flux0",
         7: "P flux1", 8: "P split2", 9: "P flux2", 10: "P flux3", 11: "P sync", 12: "P u_free", 30: "P fx_empty0",
         31: "P fx_empty1", 32: "P fx_empty2", 33: "P fx_empty3", 50: "E acc_empty", 51: "E V0", 52: "E V1",
         53: "E F0", 54: "E F1", 55: "E V2", 56: "E F2", 57: "E F3", 58: "E acc_full", 59: "E epi done"}
cells = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (55, 55, 55)
mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
elem = build_reference_element(4)
op = build_b200_operator(mesh, elem, path="tensor2")
u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
lib = _capi.load()
lib.dgm_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
op.advance(u, 1e-4, 1, use_graph=False)
op.lsrk_stage(u, op._buffers().alt, op._buffers().res, -0.4, 0.3, 1e-4)
torch.cuda.synchronize()
evs = []
for who in (0, 1):
    buf = np.zeros(2 * 4096, dtype=np.int64)
    n = lib.dgm_trace_read(buf.ctypes.data, who)
    evs.append(buf[: 2 * n].reshape(-1, 2))
ev = np.concatenate(evs)
ev = ev[np.argsort(ev[:, 1], kind="stable")]
t0 = ev[0, 1]
for tag, t in ev:
    it, code = divmod(int(tag), 100)
    if it < 4 or it > 100:
        print(f"tile {it:3d} {NAMES.get(code, code):14s} {t - t0:9d}")
last = ev[ev[:, 0] // 100 == ev[-1, 0] // 100]
print("tiles traced", int(ev[-1, 0]) // 100 + 1, "total cycles", int(ev[-1, 1] - t0))
