#!/bin/bash
# ncu A/B of SpMV kernel variants: instructions, duration, DRAM bytes, issue activity.
# usage: CFGS="c5 c2" VARS="PSELL_PAIR=0 PSELL_PAIR=1" bash scripts/ncu_ab.sh
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for c in ${CFGS:-c5}; do for v in ${VARS}; do
  env $v timeout 300 ncu --metrics $M --clock-control none -k regex:spmv_ -s 2 -c 1 --csv python scripts/prof_spmv_ab.py $c 2>/dev/null \
    | grep -E '^"[0-9]' | awk -F'","' -v c=$c -v v=$v '{printf "%s %s %-60.60s %s %s\n", c, v, $5, $13, $15}'
done; done
