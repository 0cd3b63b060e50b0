#!/bin/bash
# corrector A/B: pipelined grid kernel (default) vs EDG_CORR_PIPE=0
T=${1:-cab}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$T/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$T/pytest_gpu.log
for p in 1 0; do
  EDG_CORR_PIPE=$p timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$T/cfg2_02_p$p.json 2>&1
  EDG_CORR_PIPE=$p timeout 300 python bench.py --config cfg3 --steps 6 --warmup 3 $Q > gpurun_out/$T/cfg3_p$p.json 2>&1
  EDG_CORR_PIPE=$p timeout 300 python bench.py --config cfg1 --steps 20 $Q > gpurun_out/$T/cfg1_p$p.json 2>&1
done
B="python bench.py --config cfg2 --cfl 0.2 --steps 2 --warmup 6 $Q"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:corrector -s 6 -c 1 -o gpurun_out/$T/corr_pipe_cfg2 $B > gpurun_out/$T/ncu_corr.log 2>&1
exit 0
