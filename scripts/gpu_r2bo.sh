#!/bin/bash
# round-2 GPU pass bo: ncu --set full of the node-block kernels of the final code (configs[2] step 150, configs[3], configs[4])
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python scripts/cfg2_launch_bytes.py > gpurun_out/r2bo_cfg2_launch_bytes.json 2> gpurun_out/r2bo_lb.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 150 -c 1 \
  -o gpurun_out/r2bo_cfg2_nodes python scripts/cfg2_launch_bytes.py > gpurun_out/r2bo_ncu2.log 2>&1
timeout 600 python scripts/bench_cfg3.py --steps 8 > gpurun_out/r2bo_cfg3_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 5 -c 1 \
  -o gpurun_out/r2bo_cfg3_nodes python scripts/bench_cfg3.py --steps 8 > gpurun_out/r2bo_ncu3.log 2>&1
timeout 600 python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2bo_cfg4_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 30 -c 1 \
  -o gpurun_out/r2bo_cfg4_nodes python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2bo_ncu4.log 2>&1
ls -la gpurun_out/r2bo*; tail -n 2 gpurun_out/r2bo_ncu2.log gpurun_out/r2bo_ncu3.log gpurun_out/r2bo_ncu4.log
