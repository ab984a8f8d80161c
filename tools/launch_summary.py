"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
total device time and share per kernel (name up to the template args)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    if len(sys.argv) > 2 and sys.argv[2] == "full":
        name = r[ki][:90]
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v for _, v in agg.values())
print(f"total {tot/1e3:.1f} us over {sum(c for c,_ in agg.values())} launches (units as reported: ns)")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v/tot*100:6.2f}%  {c:6d} x {v/c/1e3:8.2f} us  {k}")
