"""Print DESIGN.md §7's results table from profiles/r02/bench_r02_full.json and the ncu summaries."""
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = os.path.join(ROOT, "profiles", "r02")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram(tag):
    rows = {r[0]: r for r in csv.reader(open(os.path.join(D, "ncu", f"ncu_{tag}_summary.csv"))) if r}
    return sum(float(rows[k][2]) * SCALE[rows[k][1]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))


def size(b):
    return "%.3g GB" % (b / 1e9) if b >= 1e9 else "%.3g MB" % (b / 1e6)


def main():
    d = json.loads(open(os.path.join(D, "bench_r02_full.json")).read())
    bw = d["roofline"]["peak"]
    rows = {"C1": ("C1 N=3, 1,512 tets, 100 steps, CUDA graph", "SIMT f32, few-tile variant", "c1")}
    for n in range(1, 10):
        kern = "SIMT f32" if n <= 2 else "tensor v1" + {5: " (42-el. tiles, 2 CTAs/SM)", 7: " (42-el. tiles)",
                                                          9: " (21-el. tiles)"}.get(n, "")
        rows["C2_N%d" % n] = ("C2 N=%d, 48k" % n, kern, "c2n%d" % n)
    rows["C3_f64"] = ("C3 N=4, 998,250, fp64", "SIMT + DMMA", "c3f64")
    rows["C4"] = ("C4 N=4, 7,986,000, 1 GPU", "tensor v1", "c4")
    rows["C5"] = ("C5 N=6, 2,058,000", "tensor v1", "c5")
    order = ["C1"] + ["C2_N%d" % n for n in range(1, 10)] + ["HEAD", "C3_f64", "C4", "C5"]
    for k in order:
        if k == "HEAD":
            v, (label, kern, tag), bold = d, ("C3 N=4, 998,250, fp32", "tensor v1", "c3"), True
        else:
            v, (label, kern, tag), bold = d["configs"][k], rows[k], False
        r = v["roofline"]
        ms = v["ms_per_step"] / 5
        cells = [label, kern, "%.4g" % ms if ms > 0.01 else "%.4f" % ms, "%.1f" % (v["value"] / 1e3),
                 "%.3f [%s]" % (r["frac"], r["bound"])]
        if bold:
            cells = ["**%s**" % c for c in cells[:1]] + cells[1:2] + ["**%s**" % c for c in cells[2:]]
        b_alg = r["hbm_term_us"] * 1e-6 * bw * 1e9
        print("| " + " | ".join(cells + ["%s vs %s" % (size(dram(tag)), size(b_alg))]) + " |")


if __name__ == "__main__":
    main()
