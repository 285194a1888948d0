python -m paper_2201_09212_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -1
timeout 1500 python scripts/bench_cfg3.py --nx 64 --max-iters 500 --cpu-iters 0 > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; tail -2 gpurun_out/cfg3.err; cat gpurun_out/cfg3.json
