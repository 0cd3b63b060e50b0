#!/bin/bash
# A/B of an environment switch on one config: ENVS="EDG_FV_L2=0 EDG_FV_L2=1" CFG="--config cfg4 --steps 20" bash tools/gpu_envab.sh <tag> [pytest -k expr]
TAG=${1:-envab}; D=gpurun_out/$TAG; mkdir -p $D
Q="--no-cpu-baseline --no-e2e --no-variant"
if [ -n "$2" ]; then
  for e in $ENVS; do env $e timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "$2" > $D/pytest_${e//=/_}.log 2>&1; echo "rc=$?" >> $D/pytest_${e//=/_}.log; done
fi
for rep in 1 2; do for e in $ENVS; do env $e timeout 300 python bench.py $CFG $Q >> $D/${e//=/_}.jsonl 2>&1; done; done
exit 0
