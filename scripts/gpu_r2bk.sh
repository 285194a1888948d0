#!/bin/bash
# round-2 GPU pass bk: ncu --set full (with source) of the packed grid kernel after the prefetch changes (configs[4])
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2bk_cfg4_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 30 -c 1 \
  -o gpurun_out/r2bk_cfg4_nodes python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2bk_ncu4.log 2>&1
tail -n 2 gpurun_out/r2bk_ncu4.log
