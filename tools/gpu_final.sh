#!/bin/bash
# full evidence run: tests, default bench line (with CPU baseline + e2e), per-config lines, reference arm
TAG=${1:-final}
mkdir -p gpurun_out/$TAG
timeout 300 python __graft_entry__.py --smoke > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$TAG/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/$TAG/bench_reference.json 2> gpurun_out/$TAG/bench_reference.err
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err
done
