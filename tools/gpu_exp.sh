#!/usr/bin/env bash
# A/B experiment batch on the GPU box:  gpurun -- bash tools/gpu_exp.sh <tag> "<cmd1>" "<cmd2>" ...
# each command's stdout/stderr go to gpurun_out/<tag>_<i>.log
set -u
T=$1; shift
mkdir -p gpurun_out
i=0
for c in "$@"; do
  timeout 900 bash -c "$c" > gpurun_out/${T}_$i.log 2>&1; echo "[$i] rc=$? : $c"; tail -3 gpurun_out/${T}_$i.log | cut -c1-400
  i=$((i+1))
done
