set -x
python -m paper_2201_09212_b200.build
timeout 900 python -m pytest tests -m gpu -q -x --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/prof_phases.py > gpurun_out/prof_phases.log 2>&1; echo rc=$?; cat gpurun_out/prof_phases.log
