#!/bin/bash
# round-2 GPU pass bx: bench with the clock sampler stopped before the e2e leg (3 runs), bench contract test, default bench (bench.py variant of that session; not kept)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 6 --no-cpu-baseline --no-subrecords 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('run $i', d['value'], [x['create_s'] for x in d['e2e']['rank0_split']], d['e2e']['value'], d['clocks'])"
done
timeout 900 python -m pytest tests/test_gpu_bench_contract.py -m gpu -q 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/r2bx_bench.json 2> gpurun_out/r2bx_bench.err; echo "bench rc $?"; cut -c1-200 gpurun_out/r2bx_bench.json
