#!/bin/bash
T=${1:-b15}; mkdir -p gpurun_out/$T
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_cfg5.json 2> gpurun_out/$T/bench_cfg5.err
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_cfg1.json 2> gpurun_out/$T/bench_cfg1.err
timeout 600 python -m pytest tests/test_gpu_solver.py -q -m gpu -k "amr or schedule" > gpurun_out/$T/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest.log
exit 0
