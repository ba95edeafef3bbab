"""Device time of to_padded / from_padded (dgm_pack / dgm_unpack) at C3, float64 natural <-> float32 padded."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_1024_b200 import build_b200_operator, build_reference_element, generate_box_mesh  # noqa: E402

dev = torch.device("cuda", 0)
mesh = generate_box_mesh((1.0, 1.0, 1.0), (55, 55, 55))
elem = build_reference_element(4)
op = build_b200_operator(mesh, elem, dtype=torch.float32, device=dev)
nat = torch.randn((6, mesh.num_elements, elem.num_nodes), dtype=torch.float64, device=dev)
pad = op.empty_state()
back = torch.empty_like(nat)
for _ in range(3):
    op.to_padded(nat, out=pad)
    op.from_padded(pad, torch.float64, out=back)
torch.cuda.synchronize()
assert torch.equal(back, nat.float().double())
for name, fn in (("pack", lambda: op.to_padded(nat, out=pad)), ("unpack", lambda: op.from_padded(pad, torch.float64, out=back))):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    nbytes = nat.numel() * 8 + pad.numel() * 4
    print(f"{name}: {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s (natural f64 + padded f32 bytes)")
