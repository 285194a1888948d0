python -m paper_2201_09212_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fem.py tests/test_gpu_scenes.py -x -q -m gpu 2>&1 | tail -1
timeout 1800 python scripts/bench_scenes.py --scenes 1024 --steps 200 2>&1 | tail -1
