#!/usr/bin/env python3
"""Per-CUDA-source-line hot spots from an ncu report (source page, CUDA + SASS).

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass --kernel-name regex:K > src.csv
    python tools/ncu_lines.py src.csv [top]
Prints the lines with the most executed warp instructions, with their warp-stall samples."""
import csv
import sys

rows = []
cur_file = None
with open(sys.argv[1]) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Line No", "Function Name") or not r[0]:
            continue
        try:
            rows.append((cur_file, int(r[0]), r[1].strip(), int(r[4]), int(r[7])))
        except (ValueError, IndexError):
            pass
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ts = sum(r[3] for r in rows) or 1
ti = sum(r[4] for r in rows) or 1
print(f"total samples {ts}, warp instructions {ti}")
for r in sorted(rows, key=lambda r: -r[4])[:top]:
    print(f"{100*r[3]/ts:5.1f}% smp {100*r[4]/ti:5.1f}% inst {r[4]/1e6:6.2f}M  {r[0]}:{r[1]}  {r[2][:80]}")
