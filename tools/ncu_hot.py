"""Top stall lines of one kernel in an ncu report:  python tools/ncu_hot.py REPORT KERNEL_REGEX [N] [cuda|sass]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
mode = sys.argv[4] if len(sys.argv) > 4 else "sass"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode, "-k", f"regex:{kern}",
                      "-c", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')]
r = list(csv.reader(io.StringIO("\n".join(lines[start[0]:]))))
h = r[0]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
rows = []
for row in r[1:]:
    try:
        v = float(row[si])
    except (ValueError, IndexError):
        continue
    top = sorted(((float(row[i] or 0), h[i]) for i in stall_cols), reverse=True)[:2]
    rows.append((v, row[0], row[src].strip()[:100], top))
tot = sum(x[0] for x in rows) or 1
for v, a, s, top in sorted(rows, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}% {a:>6} {s:100s} {' '.join(f'{t[1][6:]}={t[0]:.0f}' for t in top)}")
