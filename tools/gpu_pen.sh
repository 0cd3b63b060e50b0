#!/bin/bash
# pencil STP: gpu tests with EDG_STP_PEN=1, then A/B benches
T=${1:-pen}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
EDG_STP_PEN=1 timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/$T/pytest_pen.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$T/pytest_pen.log
for p in 1 0; do
  EDG_STP_PEN=$p timeout 300 python bench.py --cfl 0.2 $Q > gpurun_out/$T/cfg2_02_pen$p.json 2>&1
  EDG_STP_PEN=$p timeout 300 python bench.py $Q > gpurun_out/$T/cfg2_09_pen$p.json 2>&1
  EDG_STP_PEN=$p timeout 300 python bench.py --config cfg5 --steps 20 $Q > gpurun_out/$T/cfg5_pen$p.json 2>&1
  EDG_STP_PEN=$p timeout 300 python bench.py --config cfg1 --steps 20 $Q > gpurun_out/$T/cfg1_pen$p.json 2>&1
done
B="python bench.py --config cfg2 --steps 2 --warmup 6 $Q"
EDG_STP_PEN=1 $B > /dev/null 2>&1 && EDG_STP_PEN=1 ncu --set full --clock-control none --import-source on -k regex:stp_pencil -s 6 -c 1 -o gpurun_out/$T/pen_cfg2 $B > gpurun_out/$T/ncu_pen.log 2>&1
exit 0
