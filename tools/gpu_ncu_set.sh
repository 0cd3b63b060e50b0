#!/usr/bin/env bash
# ncu --set full captures of the hot kernels (one launch each, after warm-up
# steps), run on the GPU box:  gpurun -- bash tools/gpu_ncu_set.sh <tag>
set -u
T=${1:-r2}
mkdir -p gpurun_out
cap() {  # name config regex skip
  ncu --set full --import-source on --clock-control none -k "regex:$3" --launch-skip "$4" --launch-count 1 \
      -o "gpurun_out/${T}_$1" python tools/profile_step.py --config "$2" --steps 6 > "gpurun_out/${T}_$1.log" 2>&1
  echo "$1 rc=$?"
}
cap stp_cfg3 cfg3 stp_picard 3
cap corr_cfg3 cfg3 corrector 3
cap fv_cfg4 cfg4 fv_patch 3
cap stp_cfg5 cfg5 stp_picard 6
cap faces_cfg5 cfg5 faces_rusanov 6
cap restrict_cfg5 cfg5 faces_restrict 3
cap corr_cfg5 cfg5 corrector 3
