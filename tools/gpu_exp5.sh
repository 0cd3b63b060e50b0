#!/bin/bash
TAG=${1:-exp}
mkdir -p gpurun_out/$TAG
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 300 python bench.py --config cfg3 --steps 6 --warmup 2 $Q > gpurun_out/$TAG/cfg3.json 2>&1
timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$TAG/cfg2_02.json 2>&1
timeout 300 python bench.py --config cfg4 --steps 20 --warmup 3 $Q > gpurun_out/$TAG/cfg4.json 2>&1
