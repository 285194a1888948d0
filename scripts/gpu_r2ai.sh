#!/bin/bash
# round-2 GPU pass ai: serpentine slice-to-warp order in the node-block kernels
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py tests/test_gpu_fallback.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_digests.py tests/test_gpu_grid_layout.py tests/test_gpu_heightfield.py -q -x -rf > gpurun_out/r2ai_tests.log 2>&1
tail -2 gpurun_out/r2ai_tests.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-subrecords > gpurun_out/r2ai_bench.json 2> gpurun_out/r2ai_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ai_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['layout_frac'])"
timeout 600 python scripts/bench_cfg3.py --steps 20 > gpurun_out/r2ai_cfg3.json 2>> gpurun_out/r2ai.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ai_cfg3.json').read().strip().splitlines()[-1]); print('cfg3', round(d['loop_ms_total'],1), round(d['kernel']['frac'],3))"
timeout 900 python scripts/bench_cfg4.py --steps 60 > gpurun_out/r2ai_cfg4.json 2>> gpurun_out/r2ai.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ai_cfg4.json').read().strip().splitlines()[-1]); print('cfg4', round(d['loop']['loop_s'],3))"
timeout 900 python scripts/scale_projection.py --steps 2 > gpurun_out/r2ai_scale.jsonl 2>> gpurun_out/r2ai.err
python -c "
import json
for l in open('gpurun_out/r2ai_scale.jsonl'):
    d=json.loads(l); print(d['n_gpus_projected'], round(d['ms_per_run_rank'],1), round(d['projected_strong_scaling_eff'],3))"
tail -n 3 gpurun_out/r2ai.err
