#!/bin/bash
# First GPU session: build check, smoke, GPU tests, bench lines per config.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --config cfg2 --cfl 0.2 --steps 47 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_cfl02.json 2> gpurun_out/bench_cfg2_cfl02.err
