#!/bin/bash
# round-2 GPU pass v: ncu --set full of one full-size configs[4] contact-step solve (grid node-block kernel)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2v_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_iterate_nodes -s 30 -c 1 \
  -o gpurun_out/r2v_cfg4 python scripts/bench_cfg4.py --steps 32 > gpurun_out/r2v_ncu.log 2>&1
tail -c 600 gpurun_out/r2v_plain.log; tail -3 gpurun_out/r2v_ncu.log
