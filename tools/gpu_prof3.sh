#!/bin/bash
TAG=${1:-prof}
mkdir -p gpurun_out/$TAG
python tools/probe.py > gpurun_out/$TAG/probe.json 2>&1
B="python bench.py --config cfg2 --cfl 0.2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-variant"
F="python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
$B > gpurun_out/$TAG/plain_cfg2.log 2>&1 && $F > gpurun_out/$TAG/plain_cfg4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 3 -c 1 -o gpurun_out/$TAG/stp_cfg2 $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fv_patch -s 2 -c 1 -o gpurun_out/$TAG/fv_cfg4 $F > /dev/null 2>&1
echo done
