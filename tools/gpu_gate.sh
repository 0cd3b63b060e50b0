#!/bin/bash
# per-kernel event timings with the eager-step gate: small configs
T=${1:-gate}; mkdir -p gpurun_out/$T
Q="--no-cpu-baseline --no-e2e --no-variant"
for c in cfg5 cfg1 cfg4; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 $Q > gpurun_out/$T/$c.json 2>&1; done
timeout 300 python bench.py --steps 10 --warmup 3 $Q > gpurun_out/$T/cfg2.json 2>&1
B5="python bench.py --config cfg5 --steps 2 --warmup 3 $Q"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T/launches_cfg5.csv $B5 > /dev/null 2>&1
exit 0
