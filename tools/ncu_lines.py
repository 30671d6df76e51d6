"""Warp-stall samples per CUDA source line of one kernel in an ncu report.

    python tools/ncu_lines.py REPORT KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
rows, fname = [], ""
for line in out.splitlines():
    if line.startswith('"File Path"'):
        fname = line.split(",", 1)[1].strip('"').split("/")[-1]
        continue
    if line.startswith('"Function Name"') or line.startswith('"Line No"'):
        continue
    r = next(csv.reader(io.StringIO(line)))
    if len(r) > 4 and r[2] == "-":
        try:
            rows.append((float(r[4]), fname, r[0], r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows) or 1
for v, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}% {f}:{ln:5s} {src}")
