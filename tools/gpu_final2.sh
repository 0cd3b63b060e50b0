#!/bin/bash
# full evidence run + ncu: bash tools/gpu_final2.sh <tag>
TAG=${1:-final}
D=gpurun_out/$TAG; mkdir -p $D
timeout 300 python __graft_entry__.py --smoke > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err
timeout 900 python bench.py --impl reference > $D/bench_reference.json 2> $D/bench_reference.err
timeout 600 python bench.py --cfl 0.2 --no-cpu-baseline --no-variant > $D/bench_cfg2_cfl02.json 2> $D/bench_cfg2_cfl02.err
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $D/bench_$c.json 2> $D/bench_$c.err
done
Q="--no-cpu-baseline --no-e2e --no-variant"
B2="python bench.py --config cfg2 --steps 2 --warmup 3 $Q"
B4="python bench.py --config cfg4 --steps 2 --warmup 3 $Q"
B3="python bench.py --config cfg3 --steps 1 --warmup 3 $Q"
$B2 > $D/plain2.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_cfg2.csv $B2 > /dev/null 2>&1
$B4 > $D/plain4.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_cfg4.csv $B4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 3 -c 1 -o $D/stp_cfg2 $B2 > $D/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:corrector -s 3 -c 1 -o $D/corr_cfg2 $B2 > $D/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fv_patch -s 3 -c 1 -o $D/fv_cfg4 $B4 > $D/ncu3.log 2>&1
$B3 > $D/plain3.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stp_picard -s 3 -c 1 -o $D/stp_cfg3 $B3 > $D/ncu4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:corrector -s 3 -c 1 -o $D/corr_cfg3 $B3 > $D/ncu5.log 2>&1
exit 0
