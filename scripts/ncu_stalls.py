"""Warp-stall reasons per CUDA source line of an `ncu --set full` capture.
usage: python scripts/ncu_stalls.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None
rows = []
fname = "?"
tot_reason = {}
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path" and len(row) > 1:
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr and row[0].isdigit() and len(row) == len(hdr):
        try:
            s = int(row[4])
        except ValueError:
            continue
        if not s:
            continue
        reasons = {}
        for k, v in zip(hdr, row):
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    x = int(v)
                except ValueError:
                    continue
                if x:
                    reasons[k[6:]] = x
                    tot_reason[k[6:]] = tot_reason.get(k[6:], 0) + x
        rows.append((s, fname, row[0], row[1].strip()[:70], reasons))
tot = sum(r[0] for r in rows)
print("total samples", tot, " by reason:", ", ".join("%s %d" % kv for kv in sorted(tot_reason.items(), key=lambda kv: -kv[1])))
for s, f, ln, src, rs in sorted(rows, key=lambda r: -r[0])[:n]:
    top = ", ".join("%s %d" % kv for kv in sorted(rs.items(), key=lambda kv: -kv[1])[:3])
    print("%5d %5.1f%% %s:%s  %-70s  [%s]" % (s, 100.0 * s / max(tot, 1), f, ln, src, top))
