#!/bin/bash
# round-2 GPU pass bu: last check of the shipped library: smoke, node/FEM/grid/digest tests, default bench
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fem.py tests/test_gpu_grid_layout.py tests/test_gpu_fullsize_digests.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/r2bu_bench.json 2> gpurun_out/r2bu_bench.err; echo "bench rc $?"
python -c "
import json; d=json.loads(open('gpurun_out/r2bu_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['layout_frac'], d['clocks'])"
