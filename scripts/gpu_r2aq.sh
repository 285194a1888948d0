#!/bin/bash
# round-2 GPU pass aq: device memory cache (dev_alloc/dev_free) -- full -m gpu suite, e2e breakdown, bench
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r2aq_tests.log 2>&1
tail -2 gpurun_out/r2aq_tests.log
timeout 900 python scripts/e2e_cfg2_breakdown.py > gpurun_out/r2aq_e2e.json 2> gpurun_out/r2aq.err; cat gpurun_out/r2aq_e2e.json
timeout 1200 python bench.py > gpurun_out/r2aq_bench.json 2> gpurun_out/r2aq_bench.err; echo "bench rc $?"
python -c "
import json; d=json.loads(open('gpurun_out/r2aq_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['layout_frac'], d['clocks'])"
