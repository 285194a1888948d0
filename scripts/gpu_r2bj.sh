#!/bin/bash
# round-2 GPU pass bj: packed grid layout: the next issue's value offsets prefetched into shared memory (cp.async), A/B on configs[4]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grid_layout.py tests/test_gpu_fullsize_digests.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/r2bj_tests.log 2>&1; tail -n 2 gpurun_out/r2bj_tests.log
for v in default novopre; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 900 python scripts/bench_cfg4.py --steps 60 > gpurun_out/r2bj_cfg4_$v.json 2>> gpurun_out/r2bj.err
  python - <<PY
import json
d=json.loads(open('gpurun_out/r2bj_cfg4_$v.json').read().strip().splitlines()[-1])
print('$v cfg4', d.get('loop',{}).get('frac'), d.get('loop',{}).get('loop_s'))
PY
done
tail -n 3 gpurun_out/r2bj.err
