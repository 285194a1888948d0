#!/bin/bash
# round-2 GPU pass c: node-block kernel tests + full-size digests, bench, launch list, ncu of the node kernel
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_nodes.py tests/test_gpu_fallback.py tests/test_gpu_fullsize_digests.py -q > gpurun_out/r2c_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2c_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2c_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_iterate_nodes --launch-skip 150 -c 1 -o gpurun_out/r2c_nodes python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2c_ncu_full.log 2>&1
tail -3 gpurun_out/r2c_tests.log; cat gpurun_out/r2c_bench.json | head -c 1500
