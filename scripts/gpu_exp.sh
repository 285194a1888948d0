python -m paper_2201_09212_b200.build
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
timeout 600 python scripts/exp_cost.py 24,40,0,1 24,40,128,1 24,60,0,1 32,40,0,1 16,40,0,1 24,40,0,0 2>&1 | tail -6
