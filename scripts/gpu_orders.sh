#!/bin/bash
# element orders on an unstructured-numbered mesh (vertex- and element-shuffled jittered 40x40x20 box):
# stage time of the N=4 tensor kernel per internal order
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out/orders
python - > gpurun_out/orders/orders.jsonl 2>&1 <<'PY'
import json, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_0901_1024_b200 import *
torch.cuda.set_device(0)
rng = np.random.default_rng(7)
box = generate_box_mesh((1.0, 1.0, 0.5), (40, 40, 20))
v = box.vertices.copy()
inner = np.all((v > 1e-9) & (v < np.array([1, 1, 0.5]) - 1e-9), axis=1)
v[inner] += rng.uniform(-0.005, 0.005, size=(inner.sum(), 3))
perm = rng.permutation(box.num_elements)
mesh = Mesh(v, np.array([rng.permutation(r) for r in box.elements[perm]]))
elem = build_reference_element(4)
for reorder in (False, True, "morton", "greedy"):
    op = build_b200_operator(mesh, elem, reorder=reorder)
    u = op.to_padded(np.random.default_rng(1).normal(size=(6, mesh.num_elements, elem.num_nodes)))
    op.advance(u, 1e-4, 3, use_graph=False); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); op.advance(u, 1e-4, 10, use_graph=False); e.record(); torch.cuda.synchronize()
    print(json.dumps({"elements": mesh.num_elements, "reorder": str(reorder), "us_per_stage": s.elapsed_time(e) / 50 * 1e3}), flush=True)
PY
cat gpurun_out/orders/orders.jsonl
