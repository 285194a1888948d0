#!/bin/bash
# round-2 GPU pass ae: packed node-block values for single systems (grid kernel)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_heightfield.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_digests.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x -rf > gpurun_out/r2ae_tests.log 2>&1
tail -3 gpurun_out/r2ae_tests.log
timeout 600 python scripts/bench_cfg3.py --steps 20 > gpurun_out/r2ae_cfg3.json 2>> gpurun_out/r2ae.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ae_cfg3.json').read().strip().splitlines()[-1]); print('cfg3', round(d['sim_steps_per_s'],2), round(d['loop_ms_total'],1), round(d['setup_ms_total'],1), round(d['kernel']['frac'],3))"
timeout 900 python scripts/bench_cfg4.py --steps 60 > gpurun_out/r2ae_cfg4.json 2>> gpurun_out/r2ae.err
python -c "
import json; d=json.loads(open('gpurun_out/r2ae_cfg4.json').read().strip().splitlines()[-1]); print('cfg4', d['loop'])"
tail -n 3 gpurun_out/r2ae.err
