#!/bin/bash
# round-2 GPU pass j: full gpu suite, configs[4] variants subset, ncu launch list + full captures of the node kernels
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 3000 python -m pytest tests -m gpu -q -rf > gpurun_out/r2j_gputests.log 2>&1
timeout 1500 python scripts/bench_cfg4.py --scenes 4 --csv gpurun_out/r2j_cfg4_scene0.csv > gpurun_out/r2j_cfg4.json 2> gpurun_out/r2j_cfg4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2j_launches.csv python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2j_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_iterate_nodes --launch-skip 150 -c 1 -o gpurun_out/r2j_cfg2_nodes python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2j_ncu_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_iterate_nodes --launch-skip 5 -c 1 -o gpurun_out/r2j_cfg3_nodes python scripts/bench_cfg3.py --steps 7 > gpurun_out/r2j_ncu_cfg3.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_iterate_nodes --launch-skip 40 -c 1 -o gpurun_out/r2j_cfg4_nodes python scripts/bench_cfg4.py --steps 42 > gpurun_out/r2j_ncu_cfg4.log 2>&1
tail -6 gpurun_out/r2j_gputests.log; head -c 600 gpurun_out/r2j_cfg4.json
