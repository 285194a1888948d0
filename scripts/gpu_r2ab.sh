#!/bin/bash
# round-2 GPU pass ab: bench launch list of the current code (ncu gpu__time_duration, cold/serialised)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2ab_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ab_launches.csv \
  python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2ab_ncu.log 2>&1
tail -2 gpurun_out/r2ab_ncu.log
