#!/bin/bash
# persistent STP + corrector A/B (pipe vs classic) + gpu tests
T=${1:-ab3}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$T/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$T/pytest_gpu.log
for p in 1 0; do
  EDG_CORR_PIPE=$p timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$T/cfg2_02_p$p.json 2>&1
  EDG_CORR_PIPE=$p timeout 300 python bench.py --config cfg3 --steps 6 --warmup 3 $Q > gpurun_out/$T/cfg3_p$p.json 2>&1
done
timeout 300 python bench.py $Q > gpurun_out/$T/cfg2_09.json 2>&1
timeout 300 python bench.py --config cfg5 --steps 20 $Q > gpurun_out/$T/cfg5.json 2>&1
timeout 300 python bench.py --config cfg1 --steps 20 $Q > gpurun_out/$T/cfg1.json 2>&1
exit 0
