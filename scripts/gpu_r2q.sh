#!/bin/bash
# round-2 GPU pass q: resident-kernel variants (free-row warp start) on configs[1]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in default fs0 fs2; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  echo "== $v" >> gpurun_out/r2q_cfg1.log
  VFPI_LIB=$L timeout 300 python scripts/cfg1_solve.py 6 >> gpurun_out/r2q_cfg1.log 2>&1
  VFPI_LIB=$L timeout 300 python scripts/prof_phases.py > gpurun_out/r2q_phases_$v.log 2>&1
done
cat gpurun_out/r2q_cfg1.log; for v in default fs0 fs2; do echo "== $v"; head -9 gpurun_out/r2q_phases_$v.log | tail -8; done
