#!/usr/bin/env bash
# GPU evidence run (on the B200 box via gpurun, from the repo root):
#   gpurun --timeout 2400 -- bash tools/gpu_evidence.sh [pytest-args]
# 1. the GPU test suite (parity, schedule trace), 2. the default bench line
# (config 3) and the reference arm, 3. the kernel launch list of one bench
# run (ncu, clock control off).  Everything lands in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
