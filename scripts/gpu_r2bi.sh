#!/bin/bash
# round-2 GPU pass bi: the lane's node of the next slice loaded a slice ahead (all node-block kernels), A/B:
# configs[3] 20 steps, configs[4] 60 steps, configs[2] shard projection N = 1 / 8
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py tests/test_gpu_grid_layout.py tests/test_gpu_fullsize_digests.py -m gpu -q -x > gpurun_out/r2bi_tests.log 2>&1; tail -n 2 gpurun_out/r2bi_tests.log
for v in default nonodepre; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/bench_cfg3.py --steps 20 > gpurun_out/r2bi_cfg3_$v.json 2>> gpurun_out/r2bi.err
  VFPI_LIB=$L timeout 900 python scripts/bench_cfg4.py --steps 60 > gpurun_out/r2bi_cfg4_$v.json 2>> gpurun_out/r2bi.err
  VFPI_LIB=$L timeout 600 python scripts/scale_projection.py --ns 1 8 --steps 3 > gpurun_out/r2bi_$v.jsonl 2>> gpurun_out/r2bi.err
  python - <<PY
import json
for c in ('cfg3','cfg4'):
    d=json.loads(open('gpurun_out/r2bi_%s_$v.json'%c).read().strip().splitlines()[-1])
    print('$v',c,d.get('loop_ms_total'), d.get('kernel',d.get('loop',{})).get('frac'), d.get('loop',{}).get('loop_s'))
for l in open('gpurun_out/r2bi_$v.jsonl'):
    d=json.loads(l); print('$v N', d['n_gpus_projected'], round(d['ms_per_run_rank'],1))
PY
done
tail -n 3 gpurun_out/r2bi.err
