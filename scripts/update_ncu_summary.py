"""Fold ncu summary CSVs (scripts/ncu_summary.py output) into profiles/ncu_summary.json.

    python scripts/update_ncu_summary.py KEY=path/to/summary.csv [KEY=...]

KEY is "<kernel family><N>/<dtype>@<elements>", e.g. tc_stage_kernel<4>/f32@998250 -- what bench.py's
_traffic looks up (the mesh size is part of the key: traffic per launch scales with it).  Stored per launch: DRAM bytes read + written, duration, the kernel name and the source file.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_summary.json")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "s": 1e6}


def read(path):
    rows = {r[0]: r for r in csv.reader(open(path)) if r}
    name = rows["Kernel Name"][2]

    def val(metric):
        r = rows[metric]
        return float(r[2]) * SCALE[r[1]]

    return {"kernel": name,
            "dram_bytes_per_launch": int(round(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))),
            "dram_read_bytes": int(round(val("dram__bytes_read.sum"))),
            "dram_write_bytes": int(round(val("dram__bytes_write.sum"))),
            "duration_us": val("gpu__time_duration.sum"),
            "source": os.path.relpath(path, ROOT)}


def main(args):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data.setdefault("kernels", {})
    for a in args:
        key, path = a.split("=", 1)
        ent = read(path)
        if "@" in key:
            ent["elements"] = int(key.split("@", 1)[1])
        data["kernels"][key] = ent
    json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
