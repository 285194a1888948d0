#!/bin/bash
# round-2 GPU pass g: full gpu suite, bench, configs[3] 100 steps, per-launch bytes of configs[2]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 3000 python -m pytest tests -m gpu -q -rf > gpurun_out/r2g_gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
timeout 900 python scripts/bench_cfg3.py --csv gpurun_out/r2g_cfg3.csv > gpurun_out/r2g_cfg3.json 2> gpurun_out/r2g_cfg3.err
timeout 900 python scripts/bench_cfg3.py --chebyshev > gpurun_out/r2g_cfg3_cheb.json 2>> gpurun_out/r2g_cfg3.err
timeout 900 python scripts/cfg2_launch_bytes.py > gpurun_out/r2g_cfg2_launch_bytes.json 2> gpurun_out/r2g_cfg2_launch_bytes.err
tail -15 gpurun_out/r2g_gputests.log
