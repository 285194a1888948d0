#!/bin/bash
# round-2 GPU pass ax: grid node-block kernel: x gathers as two aligned 16-byte loads + issue-path loads, A/B against the previous commit
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_grid_layout.py tests/test_gpu_nodes.py tests/test_gpu_fullsize_digests.py -m gpu -q -x > gpurun_out/r2ax_tests.log 2>&1; tail -2 gpurun_out/r2ax_tests.log
for v in default hoistonly; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/bench_cfg3.py --steps 20 > gpurun_out/r2ax_cfg3_$v.json 2>> gpurun_out/r2ax.err
  VFPI_LIB=$L timeout 900 python scripts/bench_cfg4.py --steps 60 > gpurun_out/r2ax_cfg4_$v.json 2>> gpurun_out/r2ax.err
  python - <<PY
import json
for c in ('cfg3','cfg4'):
    d=json.loads(open('gpurun_out/r2ax_%s_$v.json'%c).read().strip().splitlines()[-1])
    print('$v',c,{k:d[k] for k in d if k in ('wall_s','loop_ms_total','loop_s','iter_loop_s','contact_iter_per_s')}, d.get('kernel',d.get('loop',{})).get('frac'), d.get('loop',{}).get('loop_s'))
PY
done
tail -n 3 gpurun_out/r2ax.err
