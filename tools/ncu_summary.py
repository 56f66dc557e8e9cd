"""Summarise an ncu report: key sections + raw metrics (run here, no GPU)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
sections = ('GPU Speed Of Light Throughput', 'Compute Workload Analysis', 'Memory Workload Analysis',
            'Occupancy', 'Launch Statistics', 'Warp State Statistics')
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
si, mi, vi, ui = h.index('Section Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
kn = h.index('Kernel Name')
print("kernel:", r[1][kn][:100])
for x in r[1:]:
    if x[si] in sections:
        print(f"{x[si][:24]:24s} | {x[mi]} = {x[vi]} {x[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units, v = r[0], r[1], r[2]
want = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.sum', 'smsp__inst_executed.sum', 'launch__registers_per_thread',
        'sm__sass_thread_inst_executed_op_dfma_pred_on.sum', 'sm__sass_thread_inst_executed_op_dadd_pred_on.sum',
        'sm__sass_thread_inst_executed_op_dmul_pred_on.sum', 'lts__t_sectors_op_red.sum',
        'smsp__average_warp_latency_issue_stalled_barrier', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active']
for w in want:
    if w in h:
        print(f"raw | {w} = {v[h.index(w)]} {units[h.index(w)]}")
# stall reasons
for i, name in enumerate(h):
    if name.startswith('smsp__average_warps_issue_stalled_') and name.endswith('_per_issue_active.ratio'):
        try:
            val = float(v[i])
        except ValueError:
            continue
        if val > 0.3:
            print(f"stall | {name[34:-23]} = {val:.2f}")
