#!/bin/bash
# round-2 GPU pass bs: scene kernels (template columns): x gathers two stages ahead, A/B on the configs[2] shard projection N = 1 / 8 (two rounds)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py -m gpu -q -x > gpurun_out/r2bs_tests.log 2>&1; tail -n 2 gpurun_out/r2bs_tests.log
for rnd in 1 2; do
for v in default nox2; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/scale_projection.py --ns 1 8 --steps 3 > gpurun_out/r2bs_${v}_$rnd.jsonl 2>> gpurun_out/r2bs.err
  python -c "
import json
for l in open('gpurun_out/r2bs_${v}_$rnd.jsonl'):
    d=json.loads(l); print('$v round $rnd N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
"
done
done
tail -n 3 gpurun_out/r2bs.err
