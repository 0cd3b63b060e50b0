#!/usr/bin/env bash
# Bench lines of every configuration, the reference arm, and the kernel
# launch list of the default bench (ncu, gpu__time_duration, clocks not
# locked), on the GPU box:  gpurun -- bash tools/gpu_bench_all.sh <tag>
set -u
T=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg3.json 2> gpurun_out/${T}_bench_cfg3.err; echo "cfg3 rc=$?"
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
  echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launches rc=$?"
