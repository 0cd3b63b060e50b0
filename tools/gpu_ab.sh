#!/bin/bash
# A/B of library variants built with build_lib --variant:
#   STP="base minb3" FV="base" PYTEST=1 bash tools/gpu_ab.sh <tag>
TAG=${1:-ab}
STP=${STP:-base}
FV=${FV:-}
mkdir -p gpurun_out/$TAG
Q="--no-cpu-baseline --no-e2e --no-variant"
if [ "${PYTEST:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
fi
L=paper_1806_07984_b200/_lib
libof() { if [ $1 = base ]; then echo $L/libenclavedg_b200.so; else echo $L/$1/libenclavedg_b200.so; fi; }
for v in $STP; do
  lib=$(libof $v)
  EDG_LIB=$lib timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$TAG/cfg2_02_$v.json 2>&1
  EDG_LIB=$lib timeout 300 python bench.py $Q > gpurun_out/$TAG/cfg2_09_$v.json 2>&1
  EDG_LIB=$lib timeout 300 python bench.py --config cfg5 --steps 20 $Q > gpurun_out/$TAG/cfg5_$v.json 2>&1
  [ "${CFG3:-0}" = 1 ] && EDG_LIB=$lib timeout 300 python bench.py --config cfg3 --steps 6 --warmup 3 $Q > gpurun_out/$TAG/cfg3_$v.json 2>&1
done
for v in $FV; do
  lib=$(libof $v)
  EDG_LIB=$lib timeout 300 python bench.py --config cfg4 --steps 20 $Q > gpurun_out/$TAG/cfg4_$v.json 2>&1
done
exit 0
