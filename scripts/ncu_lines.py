"""Per-source-line warp instructions and stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
fname = "?"
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        inst = int(r[7] or 0)
        samp = int(r[4] or 0)
    except ValueError:
        continue
    if inst or samp:
        agg.append((inst, samp, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot_i = sum(a[0] for a in agg)
tot_s = sum(a[1] for a in agg)
print(f"total warp instructions {tot_i:,}  samples {tot_s:,}")
for inst, samp, loc, src in sorted(agg, reverse=True)[:top]:
    print(f"{inst:>12,} {100*inst/tot_i:5.1f}%  {100*samp/max(tot_s,1):5.1f}%s  {loc:18} {src}")
