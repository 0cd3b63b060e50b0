#!/bin/bash
# bench A/B of library variants (no tests): VARS="base g3" CFGS="c02 c09 c5" bash tools/gpu_var.sh <tag> [ncu-variant]
TAG=${1:-var}; D=gpurun_out/$TAG; mkdir -p $D
L=paper_1806_07984_b200/_lib
Q="--no-cpu-baseline --no-e2e --no-variant"
for rep in 1 2; do
for v in ${VARS:-base}; do
  lib=$L/$v/libenclavedg_b200.so; [ $v = base ] && lib=$L/libenclavedg_b200.so
  for c in ${CFGS:-c02 c09 c5}; do
    case $c in
      c02) A="--cfl 0.2";; c09) A="";; c5) A="--config cfg5 --steps 20";; c3) A="--config cfg3 --steps 6 --warmup 3";;
      c1) A="--config cfg1 --steps 17";; c3f) A="--config cfg3 --steps 20 --warmup 3";; c4) A="--config cfg4 --steps 20";;
    esac
    EDG_LIB=$lib timeout 300 python bench.py $A $Q >> $D/${c}_$v.jsonl 2>&1
  done
done
done
if [ -n "$2" ]; then
  lib=$L/$2/libenclavedg_b200.so; [ $2 = base ] && lib=$L/libenclavedg_b200.so
  B="python bench.py --config cfg2 --steps 2 --warmup 6 $Q"
  EDG_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:stp_ -s 6 -c 1 -o $D/stp_$2 $B > $D/ncu_$2.log 2>&1
fi
exit 0
