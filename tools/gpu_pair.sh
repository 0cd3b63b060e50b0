#!/bin/bash
# node-pair STP A/B: correctness subset with EDG_STP_PAIR=1, then cfg2 (CFL 0.2 / 0.9) and cfg5 benches
#   VARS="base:0 base:1 p128:1" bash tools/gpu_pair.sh <tag>     (lib:pair-switch)
TAG=${1:-pair}
VARS=${VARS:-"base:0 base:1 p128:1 pm1:1"}
D=gpurun_out/$TAG; mkdir -p $D
L=paper_1806_07984_b200/_lib
libof() { if [ $1 = base ]; then echo $L/libenclavedg_b200.so; else echo $L/$1/libenclavedg_b200.so; fi; }
Q="--no-cpu-baseline --no-e2e --no-variant"
T=${TESTLIB:-base}
EDG_STP_PAIR=1 EDG_LIB=$(libof $T) timeout 900 python -m pytest tests -m gpu -q --timeout 600 \
   > $D/pytest_pair.log
for rep in 1 2; do
for v in $VARS; do
  lib=$(libof ${v%%:*}); p=${v##*:}
  EDG_STP_PAIR=$p EDG_LIB=$lib timeout 300 python bench.py --cfl 0.2 $Q >> $D/cfg2_02_${v/:/_}.jsonl 2>&1
  EDG_STP_PAIR=$p EDG_LIB=$lib timeout 300 python bench.py $Q >> $D/cfg2_09_${v/:/_}.jsonl 2>&1
  EDG_STP_PAIR=$p EDG_LIB=$lib timeout 300 python bench.py --config cfg5 --steps 20 $Q >> $D/cfg5_${v/:/_}.jsonl 2>&1
done
done
exit 0
