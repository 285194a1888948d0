#!/bin/bash
# round-2 GPU pass bp: configs[4] at spec for one rank of the 8-GPU run with the final code: variants 224..255 of the 256, 400 steps each
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2700 python scripts/bench_cfg4.py --scenes 32 --first-scene 224 > gpurun_out/r2bp_cfg4_rank7.json 2> gpurun_out/r2bp.err; echo rc $?
tail -c 900 gpurun_out/r2bp_cfg4_rank7.json; tail -n 3 gpurun_out/r2bp.err
