#!/bin/bash
# round-2 GPU pass bt: grid kernel: next stage x gathers by cp.async into a shared-memory buffer (7 warps per CTA), A/B on configs[3] / configs[4]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grid_layout.py tests/test_gpu_fullsize_digests.py tests/test_gpu_fullsize.py tests/test_gpu_nodes.py -m gpu -q -x > gpurun_out/r2bt_tests.log 2>&1; tail -n 2 gpurun_out/r2bt_tests.log
for v in default noxbuf; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 600 python scripts/bench_cfg3.py --steps 20 > gpurun_out/r2bt_cfg3_$v.json 2>> gpurun_out/r2bt.err
  VFPI_LIB=$L timeout 900 python scripts/bench_cfg4.py --steps 60 > gpurun_out/r2bt_cfg4_$v.json 2>> gpurun_out/r2bt.err
  python - <<PY
import json
for c in ('cfg3','cfg4'):
    d=json.loads(open('gpurun_out/r2bt_%s_$v.json'%c).read().strip().splitlines()[-1])
    print('$v',c,d.get('loop_ms_total'), d.get('kernel',d.get('loop',{})).get('frac'), d.get('loop',{}).get('loop_s'))
PY
done
tail -n 3 gpurun_out/r2bt.err
