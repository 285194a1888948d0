#!/bin/bash
# round-2 GPU pass k: cluster mode + inline S-contacts: node tests first, full suite, bench, cfg3, cfg4 (1 scene)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fallback.py tests/test_gpu_fullsize_digests.py -q -rf > gpurun_out/r2k_nodes.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rf > gpurun_out/r2k_gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
timeout 900 python scripts/bench_cfg3.py --csv gpurun_out/r2k_cfg3.csv > gpurun_out/r2k_cfg3.json 2> gpurun_out/r2k_cfg3.err
timeout 900 python scripts/bench_cfg4.py --scenes 1 > gpurun_out/r2k_cfg4.json 2> gpurun_out/r2k_cfg4.err
tail -4 gpurun_out/r2k_nodes.log; tail -4 gpurun_out/r2k_gputests.log
