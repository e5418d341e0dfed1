#!/bin/bash
# Dev: text digest of an ncu --set full capture: key raw metrics + the source lines holding most stall samples.
# usage: ncu_digest.sh <report.ncu-rep> <mangled kernel name> > digest.txt
rep=$1; kern=$2
echo "== $(basename $rep) : $kern"
ncu -i $rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
want=['Kernel Name','Grid Size','Block Size','gpu__time_duration.sum','launch__registers_per_thread','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','lts__t_bytes.sum','lts__throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','smsp__inst_executed.sum']
want+= [c for c in h if 'issue_stalled' in c and c.endswith('per_issue_active.ratio')]
for w in want:
    for i,c in enumerate(h):
        if c==w and v[i] not in ('0','0.000000',''): print(f'{w:90s} {v[i]} {rows[1][i] if len(rows)>2 else \"\"}')
"
echo "-- stall samples by source line"
python $(dirname $0)/../ncu_lines.py $rep $kern 25 2>&1 | tail -27
