#!/bin/bash
# Round-2 evidence in one gpurun call: bench lines for every config, the reference arm,
# ncu launch lists and --set full captures of the production SpMV kernels (summarised
# into gpurun_out/ev2/ncu_*.json; scripts/ncu_summary.py).
cd "$(dirname "$0")/.."
E=gpurun_out/ev2
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $E/gpu.txt 2>&1
for c in c1 c3 c3-e8m10 c4 c4b; do timeout -s KILL 600 python bench.py --config $c --no-pcg > $E/bench_$c.log 2>&1; done
timeout -s KILL 600 python bench.py --impl reference > $E/bench_reference_c2.log 2>&1
for c in c2 c3 c4 c4b; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv \
      --log-file $E/launches_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-pcg --no-vendor > /dev/null 2>&1
done
for c in c2 c3 c3-e8m10 c4 c4b; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"spmv_dual|spmv_pair" -s 3 -c 1 -o $E/prof_$c \
      python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-pcg --no-vendor > /dev/null 2>&1
  [ -f $E/prof_$c.ncu-rep ] && python scripts/ncu_summary.py $E/prof_$c.ncu-rep $c > $E/ncu_$c.json
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:spmv_pair -s 3 -c 1 -o $E/prof_c5 \
    python scripts/prof_c5_spmv.py > /dev/null 2>&1
[ -f $E/prof_c5.ncu-rep ] && python scripts/ncu_summary.py $E/prof_c5.ncu-rep c5 > $E/ncu_c5.json
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file $E/launches_pcg_iter.csv python scripts/pcg_iter.py 64 > /dev/null 2>&1
rm -f $E/prof_c3-e8m10.ncu-rep $E/prof_c4.ncu-rep $E/prof_c4b.ncu-rep $E/prof_c5.ncu-rep
ls -la $E
