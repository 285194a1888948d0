#!/bin/bash
# round-2 GPU pass o: configs[1] resident kernel investigation (phases, source-level ncu), scaling projection
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python scripts/prof_phases.py > gpurun_out/r2o_phases.log 2>&1
timeout 900 python scripts/scale_projection.py > gpurun_out/r2o_scale.jsonl 2> gpurun_out/r2o_scale.err
timeout 300 python scripts/cfg1_solve.py 2 > gpurun_out/r2o_cfg1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_res -s 1 -c 1 \
  -o gpurun_out/r2o_res python scripts/cfg1_solve.py 2 > gpurun_out/r2o_ncu.log 2>&1
cat gpurun_out/r2o_phases.log gpurun_out/r2o_scale.jsonl gpurun_out/r2o_cfg1.log; tail -3 gpurun_out/r2o_ncu.log
