python -m paper_2201_09212_b200.build
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
timeout 300 python scripts/prof_phases.py 2>&1 | grep -v WC
