#!/bin/bash
# round-2 GPU pass m (after container re-creation): smoke, full GPU suite, bench, launch list
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r2m_gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r2m_ref.json 2> gpurun_out/r2m_ref.err
tail -3 gpurun_out/r2m_smoke.log; tail -4 gpurun_out/r2m_gputests.log; cat gpurun_out/r2m_bench.json gpurun_out/r2m_ref.json
