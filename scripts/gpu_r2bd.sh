#!/bin/bash
# round-2 GPU pass bd: full -m gpu suite on the new scene/grid kernels + forced cluster sizes at N = 8 / 4
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r2bd_tests.log 2>&1
tail -n 2 gpurun_out/r2bd_tests.log
for cl in 0 2 4 8; do
  timeout 600 python scripts/scale_projection.py --ns 8 4 --steps 3 --cluster $cl > gpurun_out/r2bd_cl$cl.jsonl 2>> gpurun_out/r2bd.err
  python -c "
import json
for l in open('gpurun_out/r2bd_cl$cl.jsonl'):
    d=json.loads(l); print('cluster $cl N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
"
done
tail -n 3 gpurun_out/r2bd.err
