#!/bin/bash
# ncu evidence for this session's kernels: the bulk-staged K4 CSR (FP64 PCG / outer FCG
# operator) and the fused FP64 PCG iteration's launch list; the IO-CG inner iteration.
cd "$(dirname "$0")/.."
E=gpurun_out/ev3
mkdir -p $E
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:csr_spmv_bulk -s 3 -c 1 -o $E/prof_csr \
    python scripts/csr_ab.py 256 > $E/ncu_csr.log 2>&1
[ -f $E/prof_csr.ncu-rep ] && python scripts/ncu_summary.py $E/prof_csr.ncu-rep csr_bulk_f64 > $E/ncu_csr_bulk.json
NX=256 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"csr_spmv|pcg_update|xpby" -s 30 -c 30 --csv --log-file $E/launches_fp64_pcg.csv \
    python scripts/pcg64_ab.py --child > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 200 -c 60 --csv --log-file $E/launches_pcg_iter.csv python scripts/pcg_iter.py 256 > /dev/null 2>&1
rm -f $E/*.ncu-rep
ls -la $E
