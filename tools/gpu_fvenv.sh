#!/bin/bash
# cfg4 FV: default vs the runtime switches EDG_FV_MINB=2 and EDG_FV_PIPE=1 (after the volume-outer loop order)
T=${1:-fvenv}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
for r in 1 2; do
  timeout 300 python bench.py --config cfg4 --steps 20 $Q >> gpurun_out/$T/cfg4_base.jsonl 2>&1
  EDG_FV_MINB=2 timeout 300 python bench.py --config cfg4 --steps 20 $Q >> gpurun_out/$T/cfg4_minb2.jsonl 2>&1
  EDG_FV_PIPE=1 timeout 300 python bench.py --config cfg4 --steps 20 $Q >> gpurun_out/$T/cfg4_pipe.jsonl 2>&1
done
exit 0
