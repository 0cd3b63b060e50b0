#!/bin/bash
# A/B: 2-D STP derivative rows from a per-CTA shared 1/h (EDG_STP_IHS) on cfg2 (CFL 0.9 and 0.2)
T=${1:-ihs}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
L=paper_1806_07984_b200/_lib
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_gpu.log
for v in base i0 base i0; do
  lib=$L/libenclavedg_b200.so; [ $v != base ] && lib=$L/$v/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py $Q >> gpurun_out/$T/cfg2_$v.jsonl 2>&1
  EDG_LIB=$lib timeout 300 python bench.py --cfl 0.2 $Q >> gpurun_out/$T/cfg2c02_$v.jsonl 2>&1
done
exit 0
