#!/bin/bash
TAG=${1:-exp}
mkdir -p gpurun_out/$TAG
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
for th in 1 0; do
  EDG_STP_TH=$th timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$TAG/cfg2_02_th$th.json 2>&1
  EDG_STP_TH=$th timeout 300 python bench.py $Q > gpurun_out/$TAG/cfg2_09_th$th.json 2>&1
  EDG_STP_TH=$th timeout 300 python bench.py --config cfg5 --steps 20 $Q > gpurun_out/$TAG/cfg5_th$th.json 2>&1
done
