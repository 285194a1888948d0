#!/bin/bash
# round-2 GPU pass ad: weighted CTA partition of single systems (contact cost sweep on configs[3], configs[4] short)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_heightfield.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_digests.py tests/test_gpu_nodes.py tests/test_pile.py -q -x -rf > gpurun_out/r2ad_tests.log 2>&1
tail -3 gpurun_out/r2ad_tests.log
for c in 0 8 16 32 64; do
  timeout 600 python scripts/bench_cfg3.py --steps 20 --tune 11=$c > gpurun_out/r2ad_cfg3_c$c.json 2>> gpurun_out/r2ad.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2ad_cfg3_c$c.json').read().strip().splitlines()[-1]); print('cfg3 cost $c', round(d['sim_steps_per_s'],2), round(d['loop_ms_total'],1), round(d['kernel']['frac'],3))"
done
for c in 0 16 64; do
  timeout 900 python scripts/bench_cfg4.py --steps 60 --tune 11=$c > gpurun_out/r2ad_cfg4_c$c.json 2>> gpurun_out/r2ad.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2ad_cfg4_c$c.json').read().strip().splitlines()[-1]); print('cfg4 cost $c', d['loop'])"
done
tail -n 3 gpurun_out/r2ad.err
