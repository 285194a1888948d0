#!/bin/bash
# round-2 GPU pass af: packed values, pack modes 0/1/2 on configs[3] and configs[4]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_heightfield.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_digests.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x -rf > gpurun_out/r2af_tests.log 2>&1
tail -2 gpurun_out/r2af_tests.log
for m in 0 1 2; do
timeout 600 python scripts/bench_cfg3.py --steps 20 --tune 12=$m > gpurun_out/r2af_cfg3_$m.json 2>> gpurun_out/r2af.err
python -c "
import json; d=json.loads(open('gpurun_out/r2af_cfg3_$m.json').read().strip().splitlines()[-1]); print('cfg3 mode $m', round(d['loop_ms_total'],1), round(d['setup_ms_total'],1))"
timeout 900 python scripts/bench_cfg4.py --steps 60 --tune 12=$m > gpurun_out/r2af_cfg4_$m.json 2>> gpurun_out/r2af.err
python -c "
import json; d=json.loads(open('gpurun_out/r2af_cfg4_$m.json').read().strip().splitlines()[-1]); print('cfg4 mode $m', round(d['loop']['loop_s'],3), round(d['loop']['setup_s'],3))"
done
tail -n 3 gpurun_out/r2af.err
