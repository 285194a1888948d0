#!/bin/bash
# round-2 GPU pass ao: packed grid layouts put up to 3 k-steps in a ring stage (as many as its value space holds)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_grid_layout.py tests/test_gpu_nodes.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_digests.py tests/test_gpu_heightfield.py -q -x -rf > gpurun_out/r2ao_tests.log 2>&1
tail -2 gpurun_out/r2ao_tests.log
for v in default pm2 default; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  VFPI_LIB=$L timeout 900 python scripts/bench_cfg4.py --steps 60 > gpurun_out/r2ao_cfg4_$v.json 2>> gpurun_out/r2ao.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2ao_cfg4_$v.json').read().strip().splitlines()[-1]); print('cfg4 $v', round(d['loop']['loop_s'],3), d.get('kernel',{}).get('frac'))"
  VFPI_LIB=$L timeout 600 python scripts/bench_cfg3.py --steps 20 > gpurun_out/r2ao_cfg3_$v.json 2>> gpurun_out/r2ao.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2ao_cfg3_$v.json').read().strip().splitlines()[-1]); print('cfg3 $v', round(d['loop_ms_total'],1), round(d['kernel']['frac'],3))"
done
tail -n 3 gpurun_out/r2ao.err
