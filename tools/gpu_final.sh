#!/usr/bin/env bash
# Round-end style evidence on the GPU box:  gpurun -- bash tools/gpu_final.sh <tag>
# GPU test suite, smoke(), every bench line + reference arm + launch list,
# ncu --set full of the hot kernels.
set -u
T=${1:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.log
bash tools/gpu_bench_all.sh ${T}
bash tools/gpu_ncu_set.sh ${T}
# afterwards, here: bash tools/collect_evidence.sh ${T}  (copies the run into profiles/round2/)
