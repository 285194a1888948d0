#!/bin/bash
# round-2 GPU pass as: configs[2] at N = 1 on thread-block clusters (74 / 37 scenes in flight: their A fits in L2) x L2 policy of the block stream
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in default clpol1 clpol2; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  for cl in 0 4 8 2; do
    if [ $v != default ] && [ $cl = 0 ]; then continue; fi
    VFPI_LIB=$L timeout 600 python scripts/scale_projection.py --ns 1 --steps 2 --cluster $cl > gpurun_out/r2as_${v}_$cl.jsonl 2>> gpurun_out/r2as.err
    python -c "
import json
for l in open('gpurun_out/r2as_${v}_$cl.jsonl'):
    d=json.loads(l); print('$v cluster $cl', round(d['ms_per_run_rank'],1))
"
  done
done
tail -n 3 gpurun_out/r2as.err
