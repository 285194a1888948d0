#!/bin/bash
# round-2 GPU pass aj: resident kernel contact trios (three lanes per contact) vs one lane per contact
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_random.py tests/test_gpu_graphs.py tests/test_gpu_dropin_suite.py -q -x -rf > gpurun_out/r2aj_tests.log 2>&1
tail -2 gpurun_out/r2aj_tests.log
for v in default onelane; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  echo "== $v"; VFPI_LIB=$L timeout 300 python scripts/cfg1_solve.py 6 2>&1 | tail -1
done
timeout 600 python scripts/prof_phases.py > gpurun_out/r2aj_phases.log 2>&1; head -9 gpurun_out/r2aj_phases.log
