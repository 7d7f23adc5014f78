#!/usr/bin/env python
"""Per-source-line warp-stall samples from an ncu report (needs -lineinfo + --import-source).

  python tools/ncu_lines.py gpurun_out/X.ncu-rep [top_n] [kernel_regex]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
lines = {}
tot = 0
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] in ("File Path", "File Name"):
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 6 or row[0] == "":
        continue
    try:
        s = int(row[4])
    except ValueError:
        continue
    key = (fname, int(row[0]))
    lines[key] = (lines.get(key, (0, ""))[0] + s, row[1][:90])
    tot += s
print(f"total samples {tot}")
for (f, ln), (s, src) in sorted(lines.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100.0 * s / max(tot, 1):5.1f}%  {f}:{ln:<5d} {src.strip()}")
