#!/bin/bash
# GPU suite + small-config benches (corrector auto choice, eager gate)
T=${1:-small}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_gpu.log
for c in cfg1 cfg5 cfg4; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 $Q > gpurun_out/$T/$c.json 2>&1; done
for c in cfg1; do EDG_CORR_PIPE=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 $Q > gpurun_out/$T/${c}_pipe.json 2>&1; done
timeout 300 python bench.py --steps 10 --warmup 3 $Q > gpurun_out/$T/cfg2.json 2>&1
exit 0
