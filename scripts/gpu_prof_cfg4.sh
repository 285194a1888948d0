# ncu capture of the streaming iteration kernel on a configs[4] contact step
set -x
timeout 300 python scripts/bench_cfg4.py --steps 56 --max-iters 50 --cpu-iters 0 > gpurun_out/cfg4_prof_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate -s 54 -c 1 -o gpurun_out/prof_cfg4 \
  python scripts/bench_cfg4.py --steps 56 --max-iters 50 --cpu-iters 0 > gpurun_out/ncu_cfg4.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_cfg4.log
