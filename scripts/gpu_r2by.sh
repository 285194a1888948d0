#!/bin/bash
# round-2 GPU pass by: e2e construction outliers: vfpi_fem_create vs node layout split over 12 constructions (3 processes x 4)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python scripts/e2e_cfg2_breakdown.py 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for r in d['reps']: print('run $i', round(r['create_s'],4), 'fem_create', round(r['fem_create_s'],4), 'node_layout', round(r['node_layout_s'],4))"
done
