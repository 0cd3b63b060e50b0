#!/bin/bash
# quick evidence run at HEAD: smoke, GPU tests, default bench, STP ncu capture
TAG=${1:-check}
D=gpurun_out/$TAG; mkdir -p $D
timeout 300 python __graft_entry__.py --smoke > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err
Q="--no-cpu-baseline --no-e2e --no-variant"
B2="python bench.py --config cfg2 --steps 2 --warmup 6 $Q"
$B2 > $D/plain2.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 6 -c 1 -o $D/stp_cfg2 $B2 > $D/ncu1.log 2>&1
exit 0
