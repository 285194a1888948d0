#!/bin/bash
# round-2 GPU pass t: launch list of one rank's configs[2] shard at N=8 (128 scenes, 200 steps)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python scripts/scale_projection.py --ns 8 --steps 1 --warmup 1 > gpurun_out/r2t_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_launches.csv \
  python scripts/scale_projection.py --ns 8 --steps 1 --warmup 1 > gpurun_out/r2t_ncu.log 2>&1
tail -2 gpurun_out/r2t_plain.log; tail -2 gpurun_out/r2t_ncu.log
