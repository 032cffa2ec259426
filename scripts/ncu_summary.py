"""Key metrics of `ncu --set full` captures as a markdown table.
usage: python scripts/ncu_summary.py REPORT.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "HMMA/UTC subpipe %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA subpipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC/SM"),
]

print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
print("|---" * (len(KEYS) + 1) + "|")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        name = d.get("Kernel Name", "?").split("(")[0].replace("(anonymous namespace)::", "")[-48:]
        vals = []
        for k, _ in KEYS:
            v = d.get(k, "")
            vals.append((v + " " + u.get(k, "")).strip() if v else "-")
        print("| %s | %s |" % (name, " | ".join(vals)))
