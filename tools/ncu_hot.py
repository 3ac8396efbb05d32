"""Top CUDA source lines by warp-stall samples of one kernel in an ncu
--import-source report (cuda,sass correlated view): python tools/ncu_hot.py REP [top]"""
import csv
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
recs, fname = [], ""
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0].isdigit() and r[2] == "-":
        try:
            recs.append((int(r[4] or 0), fname, int(r[0]), r[1][:100]))
        except ValueError:
            pass
tot = sum(x[0] for x in recs) or 1
for smp, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{100 * smp / tot:5.1f}%  {f}:{ln:<5}  {src}")
