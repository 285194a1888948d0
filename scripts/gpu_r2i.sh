#!/bin/bash
# round-2 GPU pass i: full gpu suite, bench, configs[3] 100 steps, per-launch bytes
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fallback.py -q -rf > gpurun_out/r2i_nodes.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rf > gpurun_out/r2i_gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
timeout 900 python scripts/bench_cfg3.py --csv gpurun_out/r2i_cfg3.csv > gpurun_out/r2i_cfg3.json 2> gpurun_out/r2i_cfg3.err
timeout 900 python scripts/bench_cfg3.py --chebyshev > gpurun_out/r2i_cfg3_cheb.json 2>> gpurun_out/r2i_cfg3.err
timeout 900 python scripts/cfg2_launch_bytes.py > gpurun_out/r2i_cfg2_launch_bytes.json 2> gpurun_out/r2i_cfg2_launch_bytes.err
tail -3 gpurun_out/r2i_nodes.log; tail -12 gpurun_out/r2i_gputests.log
