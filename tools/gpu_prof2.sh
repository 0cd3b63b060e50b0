#!/bin/bash
# ncu captures of the current hot kernels: usage bash tools/gpu_prof2.sh <tag>
TAG=${1:-prof}
mkdir -p gpurun_out/$TAG
B="python bench.py --config cfg2 --cfl 0.2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variant"
F="python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
T="python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-variant"
$B > gpurun_out/$TAG/plain_cfg2.log 2>&1 && $F > gpurun_out/$TAG/plain_cfg4.log 2>&1 && $T > gpurun_out/$TAG/plain_cfg3.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_cfg2.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 2 -c 1 -o gpurun_out/$TAG/stp_cfg2 $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fv_patch -s 2 -c 1 -o gpurun_out/$TAG/fv_cfg4 $F > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 1 -c 1 -o gpurun_out/$TAG/stp_cfg3 $T > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:corrector -s 1 -c 1 -o gpurun_out/$TAG/corr_cfg3 $T > /dev/null 2>&1
echo done
