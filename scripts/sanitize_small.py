"""Tiny runs of every stage-kernel family for compute-sanitizer (racecheck / synccheck / memcheck).

One or two CTAs per launch so the sanitizers finish: the N=4 tensor kernel on 48 and 96 tets
(1 and 2 tiles of 64, one partial), N=6 tensor (1-CTA/SM kernel), N=8 (32-element tiles), N=4 fp64
and N=1 fp32 SIMT, the v2 tensor kernel at N=4 and N=3 (2 tiles), each as RHS and one LSRK4 step,
checked against the oracle.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import build_oracle_operator  # noqa: E402
from paper_0901_1024_b200 import build_b200_operator, build_reference_element, generate_box_mesh  # noqa: E402

torch.cuda.set_device(0)
cases = [((2, 2, 2), 4, torch.float32, "auto"), ((4, 2, 2), 4, torch.float32, "auto"),
         ((2, 2, 1), 6, torch.float32, "auto"), ((2, 1, 1), 8, torch.float32, "auto"),
         ((2, 2, 2), 4, torch.float64, "auto"), ((2, 2, 2), 1, torch.float32, "auto"),
         ((2, 2, 2), 4, torch.float32, "tensor2"), ((4, 2, 3), 3, torch.float32, "tensor2")]
only = sys.argv[1:]
for i, (cells, order, dtype, path) in enumerate(cases):
    if only and str(i) not in only:
        continue
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    elem = build_reference_element(order)
    op = build_b200_operator(mesh, elem, dtype=dtype, path=path)
    u0 = np.random.default_rng(i).normal(size=(6, mesh.num_elements, elem.num_nodes))
    got = op.rhs(u0)
    want = build_oracle_operator(mesh, elem).rhs(u0)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    u = op.to_padded(u0)
    op.step(u, 1e-3)
    torch.cuda.synchronize()
    print(f"case {i}: K={mesh.num_elements} N={order} {dtype} path={op.path} rhs rel L2 {err:.2e}", flush=True)
    assert err < (1e-5 if dtype == torch.float32 else 1e-12)
print("sanitize_small ok")
