# sanity: tests, smoke, default bench
set -x
python -m paper_2201_09212_b200.build
timeout 900 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?; tail -2 gpurun_out/bench_default.log
