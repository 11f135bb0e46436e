"""Stall samples per CUDA source line from an ncu report (measurement tooling):
python tools/ncu_lines.py REPORT [TOP]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
cur, agg, tot = None, {}, 0.0
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0].isdigit() and len(r) > 4 and r[2] == "-":
        try:
            s = float(r[4])
        except ValueError:
            continue
        agg[(cur, int(r[0]), r[1].strip()[:80])] = s
        tot += s
for (f, ln, s), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{ln} {s}")
