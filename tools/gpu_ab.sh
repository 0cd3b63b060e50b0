#!/bin/bash
# A/B of library variants built with build_lib --variant: bash tools/gpu_ab.sh <tag>
TAG=${1:-ab}
mkdir -p gpurun_out/$TAG
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
L=paper_1806_07984_b200/_lib
for v in base g1; do
  lib=$L/libenclavedg_b200.so; [ $v != base ] && lib=$L/$v/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$TAG/cfg2_02_$v.json 2>&1
  EDG_LIB=$lib timeout 300 python bench.py $Q > gpurun_out/$TAG/cfg2_09_$v.json 2>&1
  EDG_LIB=$lib timeout 300 python bench.py --config cfg5 --steps 20 $Q > gpurun_out/$TAG/cfg5_$v.json 2>&1
done
for v in base fvcpt1; do
  lib=$L/libenclavedg_b200.so; [ $v != base ] && lib=$L/$v/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py --config cfg4 --steps 20 $Q > gpurun_out/$TAG/cfg4_$v.json 2>&1
done
timeout 300 python bench.py --config cfg3 --steps 6 --warmup 2 $Q > gpurun_out/$TAG/cfg3_base.json 2>&1
