#!/bin/bash
# One gpurun call: build check, GPU parity tests, smoke, bench, ncu launch list + one full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p.name,p.multi_processor_count,p.L2_cache_size,p.total_memory)" >> gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "${NCU}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_run.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_c32 -s 5 -c 1 \
      -o gpurun_out/prof_spmv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_run.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/bench.log
