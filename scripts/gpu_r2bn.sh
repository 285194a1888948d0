#!/bin/bash
# round-2 GPU pass bn: final numbers of the final code -- GPU suite, smoke, bench (+ reference arm), configs[0]/[3]/[4] runs,
# scaling projection, bench launch list 
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r2bn_gputests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bn_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2bn_bench.json 2> gpurun_out/r2bn_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2bn_ref.json 2> gpurun_out/r2bn_ref.err
timeout 600 python scripts/bench_cfg0.py > gpurun_out/r2bn_cfg0.json 2> gpurun_out/r2bn_cfg.err
timeout 900 python scripts/bench_cfg3.py --csv gpurun_out/r2bn_cfg3.csv > gpurun_out/r2bn_cfg3.json 2>> gpurun_out/r2bn_cfg.err
timeout 900 python scripts/bench_cfg3.py --chebyshev > gpurun_out/r2bn_cfg3_cheb.json 2>> gpurun_out/r2bn_cfg.err
timeout 1200 python scripts/bench_cfg4.py --scenes 2 --csv gpurun_out/r2bn_cfg4.csv > gpurun_out/r2bn_cfg4.json 2>> gpurun_out/r2bn_cfg.err
timeout 900 python scripts/scale_projection.py > gpurun_out/r2bn_scale.jsonl 2> gpurun_out/r2bn_scale.err
timeout 900 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2bn_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bn_launches.csv \
  python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2bn_ncu.log 2>&1
tail -n 3 gpurun_out/r2bn_gputests.log; tail -n 2 gpurun_out/r2bn_smoke.log; cut -c1-300 gpurun_out/r2bn_bench.json
