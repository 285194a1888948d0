python -m paper_2201_09212_b200.build
timeout 300 python scripts/exp_variants.py 2>&1 | tail -9
