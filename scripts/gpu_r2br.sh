#!/bin/bash
# round-2 GPU pass br: the -m gpu suite with the test files in reverse order (order dependence / reused device memory), then smoke
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest $(ls tests/test_*.py | sort -r) -m gpu -q -rf -p no:cacheprovider > gpurun_out/r2br_tests_reverse.log 2>&1
tail -n 3 gpurun_out/r2br_tests_reverse.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
