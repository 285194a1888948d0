#!/bin/bash
# round-2 GPU pass p: resident kernel contact stream + half-sector staging + shared-reciprocal division
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I paper_2201_09212_b200/csrc \
  -o /tmp/check_ddiv3 scripts/check_ddiv3.cu && timeout 120 /tmp/check_ddiv3 > gpurun_out/r2p_ddiv3.log 2>&1
timeout 300 python scripts/cfg1_solve.py 5 > gpurun_out/r2p_cfg1.log 2>&1
timeout 600 python scripts/prof_phases.py > gpurun_out/r2p_phases.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_random.py tests/test_gpu_graphs.py -q -x -rf > gpurun_out/r2p_tests.log 2>&1
cat gpurun_out/r2p_ddiv3.log gpurun_out/r2p_cfg1.log; head -9 gpurun_out/r2p_phases.log; tail -3 gpurun_out/r2p_tests.log
