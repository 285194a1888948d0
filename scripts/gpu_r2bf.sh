#!/bin/bash
# round-2 GPU pass bf: one CTA per scene with the scene's v^(l-1) in shared memory (x gathers on chip), A/B at N = 1 / 2
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py tests/test_gpu_fullsize_digests.py -m gpu -q -x > gpurun_out/r2bf_tests.log 2>&1; tail -n 2 gpurun_out/r2bf_tests.log
for v in default noxs; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/scale_projection.py --ns 1 2 --steps 3 > gpurun_out/r2bf_$v.jsonl 2>> gpurun_out/r2bf.err
  python -c "
import json
for l in open('gpurun_out/r2bf_$v.jsonl'):
    d=json.loads(l); print('$v N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
"
done
tail -n 3 gpurun_out/r2bf.err
