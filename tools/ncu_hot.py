"""Summarise `ncu --page source --csv --print-source sass` output: per kernel,
the instructions with the most warp-stall samples and their dominant reason."""
import csv, io, sys
text = open(sys.argv[1]).read()
which = int(sys.argv[2]) if len(sys.argv) > 2 else -1
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
blocks = text.split('"Kernel Name",')[1:]
for bi, b in enumerate(blocks):
    if which >= 0 and bi != which:
        continue
    lines = b.split("\n")
    name = lines[0]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = [r for r in rows[1:] if len(r) == len(hdr)]
    total = sum(float(r[si] or 0) for r in data)
    print(f"== kernel {bi}: {name[:110]}  total samples {total:.0f}")
    agg = {}
    for r in data:
        for i in stall_cols:
            agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
    print("   reasons:", ", ".join(f"{k}={v/total*100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
    data.sort(key=lambda r: -float(r[si] or 0))
    for r in data[:top]:
        reasons = sorted(((hdr[i], float(r[i] or 0)) for i in stall_cols), key=lambda kv: -kv[1])[:2]
        print(f"   {float(r[si])/total*100:5.1f}%  {r[1].strip()[:70]:70s} {reasons}")
