"""Markdown summary of an ncu --set full report (per kernel: duration, DRAM
traffic, tensor-pipe utilisation, throughput) for profiles/."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
def col(name):
    return hdr.index(name) if name in hdr else None
want = [("duration", "gpu__time_duration.sum"),
        ("grid", "launch__grid_size"), ("regs", "launch__registers_per_thread"),
        ("dram read", "dram__bytes_read.sum"), ("dram write", "dram__bytes_write.sum"),
        ("tensor-mem active %", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 throughput %", "lts__throughput.avg.pct_of_peak_sustained_elapsed")]
# tcgen05 MMA activity: the hmma sub-pipe counts active cycles of the four
# tensor sub-units of an SM (per-SM average over all SMs); the bf16 ops-path
# counters stay 0 for tcgen05, so utilisation is derived from the cycles.
MMA = "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg"
ELAPSED = "sm__cycles_elapsed.avg"
N_SM = 148


def num(r, name):
    i = col(name)
    try:
        return float(r[i]) if i is not None else None
    except ValueError:
        return None


print(f"ncu --set full: `{rep}`\n")
extra = ["DRAM GB/s", "MMA busy % (all SMs)", "MMA busy % (SMs in grid)"]
print("| kernel | " + " | ".join([w[0] for w in want] + extra) + " |")
print("|---" * (len(want) + len(extra) + 1) + "|")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    cells = []
    for label, m in want:
        i = col(m)
        cells.append("-" if i is None else f"{r[i]} {units[i]}".strip())
    dur = num(r, "gpu__time_duration.sum")
    rd, wr = num(r, "dram__bytes_read.sum"), num(r, "dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
        units[col("dram__bytes_read.sum")], 1) if col("dram__bytes_read.sum") is not None else 1
    tscale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(units[col("gpu__time_duration.sum")], 1e-9)
    gbs = (rd + wr) * scale / (dur * tscale) / 1e9 if None not in (rd, wr, dur) else None
    mma, el, grid = num(r, MMA), num(r, ELAPSED), num(r, "launch__grid_size")
    busy = mma / (4 * el) if None not in (mma, el) and el else None
    used = busy * N_SM / min(N_SM, grid) if busy is not None and grid else None
    fmt = lambda v, f: "-" if v is None else f.format(v)  # noqa: E731
    cells += [fmt(gbs, "{:.0f}"), fmt(busy and 100 * busy, "{:.1f}"), fmt(used and 100 * used, "{:.1f}")]
    print(f"| `{name}` | " + " | ".join(cells) + " |")
