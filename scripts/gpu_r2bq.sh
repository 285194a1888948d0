#!/bin/bash
# round-2 GPU pass bq: FEM right-hand-side kernel: launch bounds / blocks per step variants (more loads in flight), configs[2] N = 1 projection, two rounds
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for rnd in 1 2; do
for v in default rhs_m3u2 rhs_m4u4 rhs_m2u4 rhs_m2u2; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/scale_projection.py --ns 1 --steps 3 > gpurun_out/r2bq_${v}_$rnd.jsonl 2>> gpurun_out/r2bq.err
  python -c "
import json
for l in open('gpurun_out/r2bq_${v}_$rnd.jsonl'):
    d=json.loads(l); print('$v round $rnd N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
"
done
done
VFPI_LIB=paper_2201_09212_b200/_variants/libvfpi_rhs_m2u4.so timeout 600 python -m pytest tests/test_gpu_fem.py -m gpu -q -x 2>&1 | tail -n 1
tail -n 3 gpurun_out/r2bq.err
