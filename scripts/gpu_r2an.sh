#!/bin/bash
# round-2 GPU pass an: ncu --set full of the resident configs[1] kernel (k_iterate_res) of the current code
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python scripts/cfg1_solve.py 1 > gpurun_out/r2an_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_iterate_res -c 1 \
  -o gpurun_out/r2an_res python scripts/cfg1_solve.py 1 > gpurun_out/r2an_ncu.log 2>&1
echo "rc $?"; tail -2 gpurun_out/r2an_plain.log; tail -3 gpurun_out/r2an_ncu.log
