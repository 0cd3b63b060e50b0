#!/usr/bin/env bash
# Copy one gpu_final.sh run (gpurun_out/<tag>_*) into profiles/round2/ and
# refresh the ncu text summaries:  bash tools/collect_evidence.sh <tag>
set -eu
T=$1; O=profiles/round2
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do cp gpurun_out/${T}_bench_$c.json $O/bench_$c.json; done
cp gpurun_out/${T}_bench_reference.json $O/bench_reference.json
cp gpurun_out/${T}_launches_cfg3.csv $O/launches_cfg3.csv
cp gpurun_out/${T}_pytest_gpu.log $O/pytest_gpu.log
cp gpurun_out/${T}_smoke.log $O/smoke.log
[ -f gpurun_out/trace_cfg5.csv ] && cp gpurun_out/trace_cfg5.csv $O/trace_cfg5_two_streams.csv
python tools/ncu_summary.py gpurun_out/${T}_stp_cfg3.ncu-rep gpurun_out/${T}_corr_cfg3.ncu-rep gpurun_out/${T}_fv_cfg4.ncu-rep \
  gpurun_out/${T}_stp_cfg5.ncu-rep gpurun_out/${T}_faces_cfg5.ncu-rep gpurun_out/${T}_restrict_cfg5.ncu-rep \
  gpurun_out/${T}_corr_cfg5.ncu-rep > $O/ncu_summary.txt
(for r in stp_cfg3 corr_cfg3 fv_cfg4; do echo "=== $r"; python tools/ncu_lines.py gpurun_out/${T}_$r.ncu-rep 25; python tools/ncu_sass_wf.py gpurun_out/${T}_$r.ncu-rep 14; done) > $O/ncu_source_lines.txt
grep -A3 "^===" $O/ncu_summary.txt | grep "===\|dram__bytes\|duration"
