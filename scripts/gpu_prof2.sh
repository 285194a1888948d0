python -m paper_2201_09212_b200.build
timeout 300 python scripts/prof_phases.py > gpurun_out/prof_phases.log 2>&1; echo rc=$?; cat gpurun_out/prof_phases.log
