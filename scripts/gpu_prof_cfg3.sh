# ncu of the single-system streaming kernel on configs[3] + launch list of a configs[4] contact step
timeout 600 python scripts/bench_cfg3.py --ncu --cpu-iters 0 > gpurun_out/cfg3_ncu_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate -s 1 -c 1 -o gpurun_out/prof_cfg3 \
  python scripts/bench_cfg3.py --ncu --cpu-iters 0 > gpurun_out/ncu_cfg3.log 2>&1; echo ncu_rc=$?
timeout 300 python scripts/bench_cfg4.py --steps 56 --max-iters 20 --cpu-iters 0 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
  python scripts/bench_cfg4.py --steps 56 --max-iters 20 --cpu-iters 0 > gpurun_out/ncu_cfg4_launch.log 2>&1; echo launch_rc=$?
