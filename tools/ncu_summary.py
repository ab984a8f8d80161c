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
        ("dram % peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("tensor-mem active %", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("tensor pipe active %", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
        ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 throughput %", "lts__throughput.avg.pct_of_peak_sustained_elapsed")]
print(f"ncu --set full: `{rep}`\n")
print("| kernel | " + " | ".join(w[0] for w in want) + " |")
print("|---" * (len(want) + 1) + "|")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    cells = []
    for label, m in want:
        i = col(m)
        cells.append("-" if i is None else f"{r[i]} {units[i]}".strip())
    print(f"| `{name}` | " + " | ".join(cells) + " |")
