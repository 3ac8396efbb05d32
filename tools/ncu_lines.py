"""Warp-stall samples per CUDA source line of an ncu report (cuda,sass source page)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, lines = None, None, []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if r and r[0] not in ("", "Function Name") and hdr:
        try:
            s = int(r[4]) if r[4] not in ("-", "") else 0
        except ValueError:
            continue
        lines.append((s, cur, r[0], r[1][:80]))
tot = sum(x[0] for x in lines) or 1
print("total samples", tot)
for s, f, ln, src in sorted(lines, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{s:7d} {100 * s / tot:5.1f}% {f}:{ln} {src}")
