#!/bin/bash
# round-2 GPU pass ay: scene kernels with a stage's x gathers issued first (template-column path) -- configs[2] shard projection N = 1 / 8 / 4, A/B against the previous commit and the start of this session
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py tests/test_gpu_fullsize_digests.py -m gpu -q -x > gpurun_out/r2bc_tests.log 2>&1; tail -n 2 gpurun_out/r2bc_tests.log
for v in default nocltcol; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/scale_projection.py --ns 8 4 2 --steps 3 > gpurun_out/r2bc_$v.jsonl 2>> gpurun_out/r2bc.err
  python -c "
import json
for l in open('gpurun_out/r2bc_$v.jsonl'):
    d=json.loads(l); print('$v N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
"
done
tail -n 3 gpurun_out/r2bc.err
