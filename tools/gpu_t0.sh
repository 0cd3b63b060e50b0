#!/bin/bash
TAG=${1:-t0}; D=gpurun_out/$TAG; mkdir -p $D
L=paper_1806_07984_b200/_lib
Q="--no-cpu-baseline --no-e2e --no-variant"
for v in base t0 t0s; do
  lib=$L/$v/libenclavedg_b200.so; [ $v = base ] && lib=$L/libenclavedg_b200.so
  EDG_LIB=$lib timeout 300 python bench.py --cfl 0.2 $Q >> $D/cfg2_02_$v.jsonl 2>&1
  EDG_LIB=$lib timeout 300 python bench.py $Q >> $D/cfg2_09_$v.jsonl 2>&1
done
B="python bench.py --config cfg2 --steps 2 --warmup 6 $Q"
for v in t0 t0s; do
  EDG_LIB=$L/$v/libenclavedg_b200.so ncu --set full --clock-control none --import-source on -k regex:stp_ -s 6 -c 1 -o $D/stp_$v $B > $D/ncu_$v.log 2>&1
done
exit 0
