#!/bin/bash
# A/B of the wide 3-D corrector CTA (EDG_CORR_WIDE) on cfg3 + the GPU suite on the new default
T=${1:-cw}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
L=paper_1806_07984_b200/_lib
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_gpu.log
for v in base w0 base w0; do
  lib=$L/libenclavedg_b200.so; [ $v != base ] && lib=$L/$v/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py --config cfg3 --steps 8 --warmup 3 $Q >> gpurun_out/$T/cfg3_$v.jsonl 2>&1
done
B3="python bench.py --config cfg3 --steps 2 --warmup 3 $Q"
ncu --set full --clock-control none --import-source on -k regex:corrector_grid -s 3 -c 1 -o gpurun_out/$T/corr_cfg3 $B3 > gpurun_out/$T/ncu.log 2>&1
exit 0
