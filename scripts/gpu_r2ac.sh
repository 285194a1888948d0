#!/bin/bash
# round-2 GPU pass aa: rhs with two blocks in flight, scene order by block radix sort
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py tests/test_gpu_fallback.py tests/test_gpu_fullsize_digests.py tests/test_gpu_scenes.py -q -x -rf > gpurun_out/r2ac_tests.log 2>&1
tail -3 gpurun_out/r2ac_tests.log
timeout 900 python scripts/scale_projection.py --steps 2 > gpurun_out/r2ac_scale.jsonl 2> gpurun_out/r2ac_scale.err
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-subrecords > gpurun_out/r2ac_bench.json 2> gpurun_out/r2ac_bench.err
python -c "
import json
for l in open('gpurun_out/r2ac_scale.jsonl'):
    d=json.loads(l); print(d['n_gpus_projected'], round(d['ms_per_run_rank'],1), round(d['projected_strong_scaling_eff'],3))
d=json.loads(open('gpurun_out/r2ac_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['e2e']['value'], d['gpu_launches'])
"; tail -n 3 gpurun_out/r2ac_scale.err gpurun_out/r2ac_bench.err
