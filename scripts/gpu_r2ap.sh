#!/bin/bash
# round-2 GPU pass ap: configs[2] e2e construction breakdown (vfpi_fem_create vs node layout)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python scripts/e2e_cfg2_breakdown.py > gpurun_out/r2ap_e2e.json 2> gpurun_out/r2ap.err; echo rc $?
cat gpurun_out/r2ap_e2e.json; tail -3 gpurun_out/r2ap.err
