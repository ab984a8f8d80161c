"""Per CUDA-source-line warp-stall summary of an ncu report
(`ncu -i rep --page source --csv --print-source cuda,sass`).
  python tools/ncu_lines.py <csv> [kernel-substring] [top]"""
import csv, io, collections, sys
text = open(sys.argv[1]).read()
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
blocks = text.split('"Function Name",')
for b in blocks[1:]:
    name = b.split("\n")[0]
    if want not in name:
        continue
    lines = b.split("\n")
    hi = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[hi:]))))
    hdr = rows[0]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    agg = collections.defaultdict(float); txt = {}
    rs = collections.defaultdict(lambda: collections.defaultdict(float))
    cur = None
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        if r[0].strip() and r[0].strip().isdigit():
            cur = int(r[0]); txt[cur] = r[1]
        if cur is None:
            continue
        try:
            v = float(r[si] or 0)
        except ValueError:
            continue
        agg[cur] += v
        for i in sc:
            try:
                rs[cur][hdr[i]] += float(r[i] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    print(f"== {name[:120]}  samples {tot:.0f}")
    for ln, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        why = sorted(rs[ln].items(), key=lambda kv: -kv[1])[:3]
        print(f"{v/tot*100:5.1f}% L{ln}: {txt.get(ln,'').strip()[:70]:70s} {[(k[6:], int(x)) for k, x in why]}")
