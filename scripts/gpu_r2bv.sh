#!/bin/bash
# round-2 GPU pass bv: e2e construction outliers: 6 e2e steps with the nvidia-smi clock sampler running through the e2e leg vs stopped before it (used a VFPI_BENCH_E2E_SAMPLER switch bench.py had during that session; removed since)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for m in 1 0 1 0; do
VFPI_BENCH_E2E_SAMPLER=$m timeout 600 python bench.py --steps 6 --warmup 3 --e2e-steps 6 --no-cpu-baseline --no-subrecords 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sampler $m', [x['create_s'] for x in d['e2e']['rank0_split']], d['e2e']['value'])"
done
