"""Export selected raw metrics of every kernel in an ncu report as CSV
(metric,unit,value per kernel).  usage: python tools/ncu_metrics.py REPORT.ncu-rep [kernel_regex]"""
import csv
import io
import re
import subprocess
import sys

KEEP = re.compile(r"^(gpu__time_duration\.sum|dram__bytes_(read|write)\.sum|smsp__inst_executed\.sum|"
                  r"sm__throughput\.avg\.pct_of_peak_sustained_elapsed|smsp__issue_active\.avg\.pct_of_peak_sustained_active|"
                  r"sm__warps_active\.avg\.pct_of_peak_sustained_active|launch__registers_per_thread|"
                  r"launch__occupancy_limit_.*|smsp__thread_inst_executed_per_inst_executed\.ratio|"
                  r"lts__t_sector_hit_rate\.pct|l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum|"
                  r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$|launch__grid_size|launch__block_size|"
                  r"dram__throughput\.avg\.pct_of_peak_sustained_elapsed|l1tex__throughput\.avg\.pct_of_peak_sustained_active|"
                  r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum|sm__inst_executed_pipe_lsu\.avg\.pct_of_peak_sustained_active)$")

rep = sys.argv[1]
kre = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
out = csv.writer(sys.stdout)
out.writerow(["kernel", "metric", "unit", "value"])
for r in rows[2:]:
    if kre and not kre.search(r[ki]):
        continue
    name = r[ki].split("(")[0]
    for i, m in enumerate(h):
        if KEEP.match(m) and r[i] not in ("", "n/a"):
            out.writerow([name, m, units[i], r[i]])
