#!/bin/bash
# ncu --set full of the STP variants on cfg2 (CFL 0.9, launch 7 = pre-NaN): VARS="lib:pair ..." bash tools/gpu_pairprof.sh <tag>
TAG=${1:-pairprof}
VARS=${VARS:-"p128:1"}
D=gpurun_out/$TAG; mkdir -p $D
L=paper_1806_07984_b200/_lib
libof() { if [ $1 = base ]; then echo $L/libenclavedg_b200.so; else echo $L/$1/libenclavedg_b200.so; fi; }
B="python bench.py --config cfg2 --steps 2 --warmup 6 --no-cpu-baseline --no-e2e --no-variant"
for v in $VARS; do
  lib=$(libof ${v%%:*}); p=${v##*:}
  EDG_STP_PAIR=$p EDG_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:stp_ -s 6 -c 1 -o $D/stp_${v/:/_} $B > $D/ncu_${v/:/_}.log 2>&1
done
exit 0
