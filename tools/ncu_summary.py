"""Summarise an ncu report (per kernel) into a short text block for profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_<name>.txt
"""
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw"], capture_output=True, text=True).stdout
kernel = None
for line in out.splitlines():
    m = re.match(r"\s+(\S.*\(\d+, \d+, \d+\)x\(\d+, \d+, \d+\).*)", line)
    if m and "Context" in line:
        kernel = m.group(1)
        print("\n== " + kernel[:160])
        continue
    parts = line.split()
    if len(parts) >= 2 and parts[0] in KEYS:
        print(f"  {parts[0]:70s} {' '.join(parts[1:])}")
