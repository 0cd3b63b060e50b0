#!/bin/bash
# A/B: 3-D STP with the derivative rows formed once per CTA and K^-1 lift from the constant bank
T=${1:-drh}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
L=paper_1806_07984_b200/_lib
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_gpu.log
for v in base old3 base old3; do
  lib=$L/libenclavedg_b200.so; [ $v != base ] && lib=$L/$v/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py --config cfg3 --steps 17 --warmup 3 $Q >> gpurun_out/$T/cfg3_$v.jsonl 2>&1
done
exit 0
