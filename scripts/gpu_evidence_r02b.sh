#!/bin/bash
# Evidence refresh at this session's production kernels: ncu --set full of one launch of
# each config's SpMV (c4 / c4b: the merged segment grid; c5: the narrow TMA kernel; K4: the
# bulk CSR kernel), launch lists of the bench steps, summarised into gpurun_out/ev4/.
cd "$(dirname "$0")/.."
E=gpurun_out/ev4
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $E/gpu.txt 2>&1
for c in c2 c3 c3-e8m10 c4 c4b; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv \
      --log-file $E/launches_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-pcg --no-vendor --no-extra > /dev/null 2>&1
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"spmv_dual|spmv_pair" -s 3 -c 1 -o $E/prof_$c \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-pcg --no-vendor --no-extra > /dev/null 2>&1
  [ -f $E/prof_$c.ncu-rep ] && python scripts/ncu_summary.py $E/prof_$c.ncu-rep $c > $E/ncu_$c.json
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:spmv_narrow -s 3 -c 1 -o $E/prof_c5 \
    python scripts/prof_c5_spmv.py > /dev/null 2>&1
[ -f $E/prof_c5.ncu-rep ] && python scripts/ncu_summary.py $E/prof_c5.ncu-rep c5 > $E/ncu_c5.json
DOT=1 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:spmv_narrow -s 3 -c 1 -o $E/prof_c5dot \
    python scripts/prof_c5_spmv.py > /dev/null 2>&1
[ -f $E/prof_c5dot.ncu-rep ] && python scripts/ncu_summary.py $E/prof_c5dot.ncu-rep c5_dot > $E/ncu_c5_dot.json
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv_bulk -s 3 -c 1 -o $E/prof_csr \
    python scripts/csr_ab.py 256 > /dev/null 2>&1
[ -f $E/prof_csr.ncu-rep ] && python scripts/ncu_summary.py $E/prof_csr.ncu-rep csr64_7pt > $E/ncu_csr64_7pt.json
rm -f $E/*.ncu-rep
ls -la $E
