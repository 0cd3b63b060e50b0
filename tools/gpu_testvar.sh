#!/bin/bash
# GPU tests of the default library, then bench A/B: VARS="base x" CFGS="c02 c09" bash tools/gpu_testvar.sh <tag> [ncu-variant]
TAG=${1:-tv}; D=gpurun_out/$TAG; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
bash tools/gpu_var.sh $TAG $2
