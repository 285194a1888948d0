python -m paper_2201_09212_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -1
timeout 300 python scripts/exp_cost.py 24,40,0,1 2>&1 | tail -1
timeout 300 python scripts/prof_phases.py 2>&1 | head -10
