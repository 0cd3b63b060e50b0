#!/bin/bash
TAG=${1:-r1c}; D=gpurun_out/$TAG; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_st.sum --csv ./tools/probes/lds_wf4 > $D/ldswf4.csv 2>&1
VARS="base map1 map2" CFGS="c3" bash tools/gpu_var.sh $TAG
exit 0
