#!/bin/bash
# ncu evidence for the SpMV kernel: launch list (share of step) + one --set full capture.
# CFG=c2|c3|c4  KREGEX=kernel regex of the production SpMV (default: dual-slice kernel)
mkdir -p gpurun_out
CFG=${CFG:-c2}
KREGEX=${KREGEX:-regex:spmv_dual|spmv_fast}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_${CFG}.csv python bench.py --config ${CFG} --steps 5 --warmup 3 --no-cpu-baseline --no-pcg > gpurun_out/ncu_launch_${CFG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "${KREGEX}" -s 3 -c 1 \
    -o gpurun_out/prof_${CFG} python bench.py --config ${CFG} --steps 5 --warmup 3 --no-cpu-baseline --no-pcg > gpurun_out/ncu_full_${CFG}.log 2>&1
echo "prof done rc=$?"
