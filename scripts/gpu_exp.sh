python -m paper_2201_09212_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-200
