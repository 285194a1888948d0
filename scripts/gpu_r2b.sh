#!/bin/bash
# round-2 GPU pass b: full gpu suite (no -x), configs[3] 100-step run
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_heightfield.py tests/test_gpu_fallback.py -q > gpurun_out/r2b_new.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2b_gputests.log 2>&1
timeout 900 python scripts/bench_cfg3.py --csv gpurun_out/r2b_cfg3.csv > gpurun_out/r2b_cfg3.json 2> gpurun_out/r2b_cfg3.err
timeout 900 python scripts/bench_cfg3.py --chebyshev > gpurun_out/r2b_cfg3_cheb.json 2>> gpurun_out/r2b_cfg3.err
tail -3 gpurun_out/r2b_gputests.log
