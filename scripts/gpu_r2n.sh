#!/bin/bash
# round-2 GPU pass n: per-config measurements of the current code (configs[0], [3], [4]) and the bench launch list
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python scripts/bench_cfg0.py > gpurun_out/r2n_cfg0.json 2> gpurun_out/r2n_cfg0.err
timeout 600 python scripts/bench_cfg0.py --chebyshev > gpurun_out/r2n_cfg0_cheb.json 2>> gpurun_out/r2n_cfg0.err
timeout 900 python scripts/bench_cfg3.py --csv gpurun_out/r2n_cfg3.csv > gpurun_out/r2n_cfg3.json 2> gpurun_out/r2n_cfg3.err
timeout 900 python scripts/bench_cfg3.py --chebyshev > gpurun_out/r2n_cfg3_cheb.json 2>> gpurun_out/r2n_cfg3.err
timeout 1200 python scripts/bench_cfg4.py --scenes 4 --csv gpurun_out/r2n_cfg4.csv > gpurun_out/r2n_cfg4.json 2> gpurun_out/r2n_cfg4.err
timeout 900 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2n_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n_launches.csv \
  python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2n_ncu.log 2>&1
cat gpurun_out/r2n_cfg0.json gpurun_out/r2n_cfg3.json gpurun_out/r2n_cfg4.json | cut -c1-600; tail -2 gpurun_out/r2n_ncu.log
