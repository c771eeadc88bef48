"""Summarise an ncu --set full capture (raw page CSV) into a markdown table:
  ncu -i X.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
M = [("time_us", "gpu__time_duration.sum"),
     ("dram_rd_MB", "dram__bytes_read.sum"),
     ("dram_wr_MB", "dram__bytes_write.sum"),
     # tcgen05-aware: tensor-memory (TMEM) activity of the UTC (tcgen05) pipe, and
     # the tcgen05.mma instruction count; the legacy pipe_tensor counter only sees
     # mma.sync (HMMA) and reads ~1-5 % for tcgen05 kernels
     ("tcgen05_tmem_pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
     ("utcmma_inst", "smsp__sass_inst_executed_op_utcmma.sum"),
     ("hmma_pct", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
     ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
     ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
     ("regs", "launch__registers_per_thread"),
     ("warps_pct", "sm__warps_active.avg.pct_of_peak_sustained_active")]
M = [(k, m) for k, m in M if m in col]


def conv(v, u, key):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if key == "time_us":
        x *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
    if key.endswith("_MB"):
        x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1, "GB": 1e3}.get(u, 1)
    return round(x, 2)


print("| kernel | grid | block | " + " | ".join(k for k, _ in M) + " |")
print("|---" * (3 + len(M)) + "|")
for r in rows[2:]:
    name = r[col["Kernel Name"]][:60]
    vals = [conv(r[col[m]], units[col[m]], k) for k, m in M]
    print(f"| {name} | {r[col['Grid Size']]} | {r[col['Block Size']]} | " + " | ".join(str(v) for v in vals) + " |")
