#!/bin/bash
# ncu --set full of the STP (cfg2, CFL 0.9, pre-NaN launch) and the corrector
mkdir -p gpurun_out/prof5
B="python bench.py --config cfg2 --steps 2 --warmup 6 --no-cpu-baseline --no-e2e --no-variant"
$B > gpurun_out/prof5/plain.json 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 6 -c 1 -o gpurun_out/prof5/stp_cfg2 $B > gpurun_out/prof5/ncu_stp.log 2>&1 ;
ncu --set full --clock-control none --import-source on -k regex:corrector -s 6 -c 1 -o gpurun_out/prof5/corr_cfg2 $B > gpurun_out/prof5/ncu_corr.log 2>&1 ;
exit 0
