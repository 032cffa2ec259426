"""Warp-stall samples per CUDA source line (kernel built with -lineinfo).
usage: python scripts/ncu_lines.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res = []
fname = "?"
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path" and len(row) > 1:
        fname = row[1].split("/")[-1]
        continue
    if row[0].isdigit() and len(row) > 4:
        try:
            s = int(row[4])
        except ValueError:
            continue
        if s:
            res.append((s, fname, row[0], row[1].strip()[:100]))
tot = sum(r[0] for r in res)
print("total samples", tot)
for s, f, ln, src in sorted(res, reverse=True)[:n]:
    print("%6d %5.1f%%  %s:%s  %s" % (s, 100.0 * s / max(tot, 1), f, ln, src))
