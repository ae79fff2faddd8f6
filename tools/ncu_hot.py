#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from an ncu report (source page).

    python tools/ncu_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
inot = hdr.index("Warp Stall Sampling (Not-issued Samples)")
iex = hdr.index("Instructions Executed")
recs = []
for idx, r in enumerate(rows[1:]):
    try:
        recs.append((int(r[iall] or 0), int(r[inot] or 0), int(r[iex] or 0), idx, r[ia], r[isrc].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in recs)
print(f"total samples {tot}")
for s_all, s_not, ex, idx, addr, src in sorted(recs, reverse=True)[:top]:
    print(f"{s_all:8d} {100.0 * s_all / max(1, tot):5.1f}%  not-issued {s_not:8d}  exec {ex:10d}  #{idx:5d}  {src[:90]}")
