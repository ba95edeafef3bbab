"""Pinned host <-> device copy rates for the e2e leg's buffer size (C3 fp32 natural state)."""
import json
import torch

n = 6 * 998250 * 35  # C3 natural state, fp32
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
gb = n * 4 / 1e9


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


big = torch.empty(1 << 30, dtype=torch.float32, device="cuda")  # 4.3 GB: HBM-bound filler work
s3 = torch.cuda.Stream()


def both_busy():
    cur = torch.cuda.current_stream()
    s3.wait_stream(cur)
    with torch.cuda.stream(s3):
        for _ in range(8):  # ~8 x 1.2 ms of HBM traffic, like one LSRK4 step of the stage kernel
            big.mul_(1.0)
    both()
    cur.wait_stream(s3)


h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
bi = timed(both)
busy = timed(both_busy)
fill = timed(lambda: [big.mul_(1.0) for _ in range(8)])
print(json.dumps({"bytes": n * 4, "h2d_ms": h2d, "h2d_gbs": gb / h2d * 1e3, "d2h_ms": d2h, "d2h_gbs": gb / d2h * 1e3,
                  "bidir_ms": bi, "bidir_gbs_each": gb / bi * 1e3,
                  "bidir_with_hbm_work_ms": busy, "hbm_work_alone_ms": fill}))
