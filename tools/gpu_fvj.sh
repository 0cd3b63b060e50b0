#!/bin/bash
# A/B of the FV loop order (EDG_FV_JOUTER) on cfg4 + the FV parity tests on the new default
T=${1:-fvj}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
L=paper_1806_07984_b200/_lib
timeout 900 python -m pytest tests -m gpu -q -k "fv or FV or cfg4 or patch or boundary" > gpurun_out/$T/pytest_fv.log 2>&1; echo "rc=$?" >> gpurun_out/$T/pytest_fv.log
for v in base j0 base j0; do
  lib=$L/libenclavedg_b200.so; [ $v != base ] && lib=$L/$v/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py --config cfg4 --steps 20 $Q >> gpurun_out/$T/cfg4_$v.jsonl 2>&1
done
B4="python bench.py --config cfg4 --steps 2 --warmup 3 $Q"
ncu --set full --clock-control none --import-source on -k regex:fv_ -s 3 -c 1 -o gpurun_out/$T/fv_j1 $B4 > gpurun_out/$T/ncu.log 2>&1
exit 0
