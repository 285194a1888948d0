python -m paper_2201_09212_b200.build
timeout 900 python -m pytest tests/test_gpu_fem.py tests/test_gpu_parity.py -m gpu -q -x --tb=short -p no:cacheprovider 2>&1 | tail -8
