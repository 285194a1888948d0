#!/bin/bash
# round-2 GPU pass bb: ncu --set full (with source) of the configs[2] scene kernel after the gather changes (step 150)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python scripts/cfg2_launch_bytes.py > gpurun_out/r2bb_cfg2_launch_bytes.json 2> gpurun_out/r2bb_lb.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 150 -c 1 \
  -o gpurun_out/r2bb_cfg2_nodes python scripts/cfg2_launch_bytes.py > gpurun_out/r2bb_ncu2.log 2>&1
ls -la gpurun_out/r2bb*; tail -n 2 gpurun_out/r2bb_ncu2.log
