#!/bin/bash
# ncu evidence: launch list + one --set full capture per hot kernel (1 GPU).
set -x
mkdir -p gpurun_out
B="python bench.py --config cfg2 --cfl 0.2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variant"
F="python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
T="python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_cfg2.log 2>&1 && $F > gpurun_out/plain_cfg4.log 2>&1 && $T > gpurun_out/plain_cfg3.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_l2.log 2>&1 ;
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 2 -c 1 -o gpurun_out/prof_stp_cfg2 $B > gpurun_out/ncu_stp2.log 2>&1 ;
ncu --set full --clock-control none --import-source on -k regex:corrector -s 2 -c 1 -o gpurun_out/prof_corr_cfg2 $B > gpurun_out/ncu_corr2.log 2>&1 ;
ncu --set full --clock-control none --import-source on -k regex:fv_patch -s 2 -c 1 -o gpurun_out/prof_fv_cfg4 $F > gpurun_out/ncu_fv.log 2>&1 ;
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 1 -c 1 -o gpurun_out/prof_stp_cfg3 $T > gpurun_out/ncu_stp3.log 2>&1 ;
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
