python -m paper_2201_09212_b200.build
timeout 900 python -m pytest tests -m gpu -q -x --tb=short -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/exp_variants.py 2>&1 | tail -5
timeout 300 python scripts/bench_scenes_kernel.py --reps 2 2>&1 | tail -1
