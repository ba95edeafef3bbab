"""Quick v2 kernel check on tiny meshes (run with DGM_LIB=.../libdgm_trace.so to turn hangs into traps)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import build_oracle_operator  # noqa: E402
from paper_0901_1024_b200 import build_b200_operator, build_reference_element, generate_box_mesh  # noqa: E402
from paper_0901_1024_b200 import _capi  # noqa: E402

torch.cuda.set_device(0)
for cells, n in [((1, 1, 1), 4), ((2, 2, 2), 4), ((4, 3, 3), 4), ((3, 3, 3), 3), ((2, 2, 2), 2), ((2, 2, 2), 1)]:
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, path="tensor2")
    u0 = np.random.default_rng(0).normal(size=(6, mesh.num_elements, elem.num_nodes))
    try:
        got = op.rhs(u0)
        torch.cuda.synchronize()
    except Exception as exc:
        print("FAILED", cells, n, exc, flush=True)
        lib = _capi.load()
        if hasattr(lib, "dgm_hang_read"):
            h = (ctypes.c_uint * 8)()
            lib.dgm_hang_read(h)
            print("hang record (flag, block, thread, mbar smem addr, parity):", list(h)[:5], flush=True)
        raise
    want = build_oracle_operator(mesh, elem).rhs(u0)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"cells={cells} N={n} K={mesh.num_elements}: rhs rel L2 {err:.3e}", flush=True)
