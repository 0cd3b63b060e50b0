#!/bin/bash
# round-1 evidence: launch lists + full captures of the hot kernels (1 GPU)
TAG=${1:-prof}
mkdir -p gpurun_out/$TAG
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-variant"
B2="python bench.py --cfl 0.2 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-variant"
F="python bench.py --config cfg4 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
T="python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-variant"
$B > gpurun_out/$TAG/plain_cfg2.log 2>&1 && $B2 > gpurun_out/$TAG/plain_cfg2_02.log 2>&1 && $F > gpurun_out/$TAG/plain_cfg4.log 2>&1 && $T > gpurun_out/$TAG/plain_cfg3.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_cfg2.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_cfg4.csv $F > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 4 -c 1 -o gpurun_out/$TAG/stp_cfg2 $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 4 -c 1 -o gpurun_out/$TAG/stp_cfg2_02 $B2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:corrector -s 4 -c 1 -o gpurun_out/$TAG/corr_cfg2 $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fv_patch -s 4 -c 1 -o gpurun_out/$TAG/fv_cfg4 $F > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 1 -c 1 -o gpurun_out/$TAG/stp_cfg3 $T > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:corrector -s 1 -c 1 -o gpurun_out/$TAG/corr_cfg3 $T > /dev/null 2>&1
echo done
