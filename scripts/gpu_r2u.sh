#!/bin/bash
# round-2 GPU pass u: CTAs per scene at N=4 / N=8 shard sizes (longest-first order on)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for c in 1 2 4 8; do
  timeout 600 python scripts/scale_projection.py --ns 4 8 --cluster $c --steps 2 > gpurun_out/r2u_c$c.jsonl 2>> gpurun_out/r2u.err
done
for c in 1 2 4 8; do python -c "
import json,sys
for l in open('gpurun_out/r2u_c$c.jsonl'):
    d=json.loads(l); print('cluster $c N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
"; done; tail -3 gpurun_out/r2u.err
