#!/bin/bash
# Round evidence in one gpurun call: GPU tests, smoke, bench lines for every config, the
# reference arm, ncu launch lists and --set full captures of the production SpMV kernels.
mkdir -p gpurun_out/ev
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/ev/gpu.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/ev/bench_c2.log 2>&1
for c in c1 c3 c4; do timeout -s KILL 600 python bench.py --config $c --no-pcg > gpurun_out/ev/bench_$c.log 2>&1; done
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/ev/bench_reference.log 2>&1
for c in c2 c3 c4; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/ev/launches_$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-pcg > /dev/null 2>&1
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:spmv_dual -s 3 -c 1 -o gpurun_out/ev/prof_c2 \
    python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --no-pcg > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:spmv_dual -s 3 -c 1 -o gpurun_out/ev/prof_c3 \
    python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-pcg > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:spmv_dual -s 3 -c 1 -o gpurun_out/ev/prof_c4 \
    python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-pcg > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:spmv_pair -s 3 -c 1 -o gpurun_out/ev/prof_c5 \
    python scripts/prof_c5_spmv.py > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/ev/launches_pcg_iter.csv python scripts/pcg_iter.py 64 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv_pipe -s 3 -c 1 -o gpurun_out/ev/prof_csr \
    python scripts/csr_ab.py > /dev/null 2>&1
timeout -s KILL 300 python scripts/iocg_kernels.py > gpurun_out/ev/iocg_kernels.txt 2>&1
timeout -s KILL 300 python scripts/pcg64_kernels.py > gpurun_out/ev/pcg64_kernels.txt 2>&1
timeout -s KILL 300 python scripts/sell_iocg.py > gpurun_out/ev/sell_iocg.txt 2>&1
PYTHONPATH=$PWD:$PWD/scripts timeout -s KILL 300 python scripts/accuracy_sell.py > gpurun_out/ev/accuracy_sell.txt 2>&1
PYTHONPATH=$PWD:$PWD/scripts timeout -s KILL 300 python scripts/cusparse_ab.py > gpurun_out/ev/cusparse_ab.txt 2>&1
timeout -s KILL 200 python scripts/csr_ab.py > gpurun_out/ev/csr_time.txt 2>&1
timeout -s KILL 300 python scripts/spmv_time.py c2 c3 c5 > gpurun_out/ev/spmv_time.txt 2>&1
timeout -s KILL 200 python scripts/upload_probe.py > gpurun_out/ev/upload_probe.txt 2>&1
# summaries of every capture; only the c2 / c5 reports travel back (gpurun_out is capped at 64 MiB)
for r in c2 c3 c4 c5 csr; do
  [ -f gpurun_out/ev/prof_$r.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/ev/prof_$r.ncu-rep $r > gpurun_out/ev/ncu_$r.json
done
rm -f gpurun_out/ev/prof_c3.ncu-rep gpurun_out/ev/prof_c4.ncu-rep gpurun_out/ev/prof_csr.ncu-rep
tail -2 gpurun_out/ev/pytest_gpu.log; tail -1 gpurun_out/ev/smoke.log
