#!/bin/bash
# One gpurun call: GPU parity tests, smoke, default bench, ncu evidence for c2 and c3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "${NCU}" ]; then
  for c in ${NCU}; do CFG=$c bash scripts/gpu_prof.sh; done
fi
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/bench.log | cut -c1-600
