"""Per-source-line instruction / stall-sample shares of one kernel from an ncu report
(ncu --page source --print-source cuda,sass).  Usage: ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ii = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
src = {}
for r in rows:
    if len(r) <= ii or r[0] in ("Line No", "File Path", "Function Name"):
        continue
    if r[0]:
        cur = (int(r[0]), r[1].strip())
        src.setdefault(cur, [0.0, 0.0])
        continue
try:
    pass
except Exception:
    pass
# second pass: the line rows carry the aggregate of their SASS rows
lines = []
for r in rows:
    if len(r) > ii and r[0] not in ("", "Line No", "File Path", "Function Name"):
        try:
            lines.append((int(r[0]), r[1].strip(), float(r[ii] or 0), float(r[si] or 0)))
        except ValueError:
            pass
ti = sum(x[2] for x in lines) or 1.0
ts = sum(x[3] for x in lines) or 1.0
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for ln, s, i, st in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{ln:5d} {100 * i / ti:5.1f}% inst {100 * st / ts:5.1f}% stall  {s[:110]}")
