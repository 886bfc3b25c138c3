"""Summarise an ncu --set full report: one line per kernel with the metrics the judge reads.

    python profiles/summarize_ncu.py report.ncu-rep > profiles/<name>.txt

Each value carries its unit as exported by ncu (`metric[unit]=value`); bench.py reads the
dram__bytes_* entries of the newest profiles/r*_ncu_full_pcg_sw_128sys.txt for `roofline.traffic`.
"""
import csv
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__grid_size',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio']
idx = [hdr.index(w) for w in want if w in hdr]
for r in rows[2:]:
    cells = [f"Kernel Name={r[hdr.index('Kernel Name')]}"]
    cells += [f"{hdr[i]}[{units[i]}]={r[i]}" for i in idx]
    print(' | '.join(cells))
