#!/bin/bash
TAG=${1:-perm3}; D=gpurun_out/$TAG; mkdir -p $D
L=paper_1806_07984_b200/_lib
EDG_LIB=$L/perm3/libenclavedg_b200.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "cfg3 or 3d or euler3 or stp" > $D/pytest_perm3.log 2>&1; echo "rc=$?" >> $D/pytest_perm3.log
VARS="base perm3" CFGS="c3" bash tools/gpu_var.sh $TAG
Q="--no-cpu-baseline --no-e2e --no-variant"
B3="python bench.py --config cfg3 --steps 1 --warmup 3 $Q"
EDG_LIB=$L/perm3/libenclavedg_b200.so ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 3 -c 1 -o $D/stp_cfg3_perm3 $B3 > $D/ncu.log 2>&1
exit 0
