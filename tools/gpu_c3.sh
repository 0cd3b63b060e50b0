#!/bin/bash
T=${1:-c3}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
for p in 1 0; do
  EDG_CORR_PIPE=$p timeout 300 python bench.py --config cfg3 --steps 6 --warmup 3 $Q > gpurun_out/$T/cfg3_p$p.json 2>&1
done
timeout 600 python -m pytest tests/test_gpu_variants.py -q -m gpu > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
exit 0
