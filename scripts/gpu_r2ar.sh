#!/bin/bash
# round-2 GPU pass ar: re-entry validation (container re-created): full -m gpu suite, smoke, bench, reference arm
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r2ar_tests.log 2>&1
tail -2 gpurun_out/r2ar_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ar_smoke.log 2>&1; tail -1 gpurun_out/r2ar_smoke.log
timeout 1200 python bench.py > gpurun_out/r2ar_bench.json 2> gpurun_out/r2ar_bench.err; echo "bench rc $?"
python -c "
import json; d=json.loads(open('gpurun_out/r2ar_bench.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['layout_frac'], d['clocks'])"
timeout 900 python bench.py --impl reference > gpurun_out/r2ar_ref.json 2> gpurun_out/r2ar_ref.err; echo "ref rc $?"; tail -c 600 gpurun_out/r2ar_ref.json
