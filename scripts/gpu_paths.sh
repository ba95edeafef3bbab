#!/bin/bash
# path comparison per config: C1 (graph path) and the C2 order sweep on the SIMT and tensor kernels
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
O=gpurun_out/paths; mkdir -p $O
python - > $O/paths.jsonl 2> $O/paths.err <<'PY'
import json, sys, time, torch
sys.path.insert(0, '.')
from paper_0901_1024_b200 import *
torch.cuda.set_device(0)
def run(cells, n, path, steps, graph):
    mesh = generate_box_mesh((1.0, 1.0, 1.0), cells)
    elem = build_reference_element(n)
    op = build_b200_operator(mesh, elem, path=path)
    dt = stable_dt(mesh, op.geometry, n)
    u = op.to_padded(CavityMode(1, 1, 1, (1.0, 1.0, 1.0)).evaluate(map_nodes(mesh, elem), 0.0))
    op.advance(u, dt, 5, use_graph=graph); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); op.advance(u, dt, steps, use_graph=graph); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / steps / 5 * 1e3, op.path
for path in ("simt", "tensor", "tensor2"):
    try:
        us, p = run((6, 6, 7), 3, path, 200, True)
        print(json.dumps({"cfg": "C1", "order": 3, "path": p, "us_per_stage": us}), flush=True)
    except Exception as ex:
        print(json.dumps({"cfg": "C1", "path": path, "error": str(ex)}), flush=True)
for n in range(1, 10):
    for path in ("simt", "tensor", "tensor2"):
        try:
            us, p = run((20, 20, 20), n, path, 20, False)
            print(json.dumps({"cfg": "C2", "order": n, "path": p, "us_per_stage": us}), flush=True)
        except Exception as ex:
            print(json.dumps({"cfg": "C2", "order": n, "path": path, "error": str(ex)[:80]}), flush=True)
PY
cat $O/paths.jsonl
