#!/bin/bash
# round-2 GPU pass y: L2 keep fraction of the streamed node blocks (experiment) at N = 8 / 4 shard sizes
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in default keep05 keep08 keep10; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/scale_projection.py --ns 8 4 1 --steps 2 > gpurun_out/r2y_$v.jsonl 2>> gpurun_out/r2y.err
  python -c "
import json
for l in open('gpurun_out/r2y_$v.jsonl'):
    d=json.loads(l); print('$v N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
"
done
tail -n 3 gpurun_out/r2y.err
