#!/bin/bash
TAG=${1:-quad}; D=gpurun_out/$TAG; mkdir -p $D
L=paper_1806_07984_b200/_lib
Q="--no-cpu-baseline --no-e2e --no-variant"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
for v in ${VARS:-base qns}; do
  lib=$L/$v/libenclavedg_b200.so; [ $v = base ] && lib=$L/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py --cfl 0.2 $Q >> $D/cfg2_02_$v.jsonl 2>&1
  EDG_LIB=$lib timeout 300 python bench.py $Q >> $D/cfg2_09_$v.jsonl 2>&1
  EDG_LIB=$lib timeout 300 python bench.py --config cfg5 --steps 20 $Q >> $D/cfg5_$v.jsonl 2>&1
  EDG_LIB=$lib timeout 300 python bench.py --config cfg1 --steps 17 $Q >> $D/cfg1_$v.jsonl 2>&1
done
B="python bench.py --config cfg2 --steps 2 --warmup 6 $Q"
ncu --set full --clock-control none --import-source on -k regex:stp_ -s 6 -c 1 -o $D/stp_base $B > $D/ncu_base.log 2>&1
exit 0
