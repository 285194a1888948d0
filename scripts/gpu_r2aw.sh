#!/bin/bash
# round-2 GPU pass aw: ncu --set full (with source) of the grid node-block kernel after the issue-path change (configs[3], configs[4])
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python scripts/bench_cfg3.py --steps 8 > gpurun_out/r2aw_cfg3_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 5 -c 1 \
  -o gpurun_out/r2aw_cfg3_nodes python scripts/bench_cfg3.py --steps 8 > gpurun_out/r2aw_ncu3.log 2>&1
timeout 600 python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2aw_cfg4_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 30 -c 1 \
  -o gpurun_out/r2aw_cfg4_nodes python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2aw_ncu4.log 2>&1
ls -la gpurun_out/r2aw*; tail -n 2 gpurun_out/r2aw_ncu4.log
