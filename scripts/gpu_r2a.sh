#!/bin/bash
# round-2 first GPU pass: new tests, full gpu suite, bench (configs[2])
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fallback.py -x -q > gpurun_out/r2a_fallback.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1
tail -3 gpurun_out/r2a_bench.log
