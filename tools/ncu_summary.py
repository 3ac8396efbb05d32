"""Key counters of an ncu --set full report, one line per kernel launch."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = {
    "Kernel Name": "kernel",
    "gpu__time_duration.sum": "time",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor%",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "bank_conf",
}
idx = {v: hdr.index(k) for k, v in want.items() if k in hdr}
units = rows[1]
for r in rows[2:]:
    print("  ".join(f"{k}={r[i][:40]}{'' if k == 'kernel' else units[i][:6]}" for k, i in idx.items()))
