#!/bin/bash
T=${1:-fvab}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$T/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$T/pytest_gpu.log
for p in 1 0; do
  EDG_FV_PIPE=$p timeout 300 python bench.py --config cfg4 --steps 20 $Q > gpurun_out/$T/cfg4_p$p.json 2>&1
done
timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$T/cfg2_02.json 2>&1
timeout 300 python bench.py --config cfg3 --steps 6 --warmup 3 $Q > gpurun_out/$T/cfg3.json 2>&1
B4="python bench.py --config cfg4 --steps 2 --warmup 3 $Q"
$B4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fv_ -s 3 -c 1 -o gpurun_out/$T/fv_pipe $B4 > gpurun_out/$T/ncu.log 2>&1
exit 0
