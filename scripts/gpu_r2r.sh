#!/bin/bash
# round-2 GPU pass r: resident kernel (half-sector staging, byte-offset maps, shared-reciprocal division) + variant
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in default fs0; do
  if [ $v = default ]; then L=""; else L=paper_2201_09212_b200/_variants/libvfpi_$v.so; fi
  echo "== $v" >> gpurun_out/r2r_cfg1.log
  VFPI_LIB=$L timeout 300 python scripts/cfg1_solve.py 6 >> gpurun_out/r2r_cfg1.log 2>&1
done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_random.py tests/test_gpu_graphs.py -q -x -rf > gpurun_out/r2r_tests.log 2>&1
cat gpurun_out/r2r_cfg1.log; tail -3 gpurun_out/r2r_tests.log
