#!/bin/bash
# Iteration loop on the GPU box: GPU tests, then short bench lines per config.
# usage: bash tools/gpu_iter.sh [tag] [--no-tests]
TAG=${1:-iter}
mkdir -p gpurun_out/$TAG
if [ "$2" != "--no-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/$TAG/bench_cfg2.json 2> gpurun_out/$TAG/bench_cfg2.err
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/$TAG/bench_cfg3.json 2> gpurun_out/$TAG/bench_cfg3.err
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_cfg4.json 2> gpurun_out/$TAG/bench_cfg4.err
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/$TAG/bench_cfg5.json 2> gpurun_out/$TAG/bench_cfg5.err
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline --no-variant > gpurun_out/$TAG/bench_cfg1.json 2> gpurun_out/$TAG/bench_cfg1.err
