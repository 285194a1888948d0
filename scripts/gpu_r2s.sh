#!/bin/bash
# round-2 GPU pass s: longest-first scene order + >= 1.5-wave cluster sizing (scene batches)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python scripts/scale_projection.py > gpurun_out/r2s_scale.jsonl 2> gpurun_out/r2s_scale.err
timeout 2400 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py tests/test_gpu_fallback.py tests/test_gpu_fullsize_digests.py tests/test_gpu_scenes.py -q -x -rf > gpurun_out/r2s_tests.log 2>&1
python -c "
import json
for l in open('gpurun_out/r2s_scale.jsonl'):
    d=json.loads(l); print(d['n_gpus_projected'], round(d['ms_per_run_rank'],1), round(d['projected_strong_scaling_eff'],3))
"; tail -3 gpurun_out/r2s_scale.err; tail -3 gpurun_out/r2s_tests.log
