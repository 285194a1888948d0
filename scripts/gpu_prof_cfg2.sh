# ncu of the scene-batch kernel (TMA-ring SELL stream) on the configs[2]-shaped batch
timeout 300 python scripts/bench_scenes_kernel.py --reps 1 > gpurun_out/cfg2_kernel_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate -s 1 -c 1 -o gpurun_out/prof_cfg2 \
  python scripts/bench_scenes_kernel.py --reps 1 > gpurun_out/ncu_cfg2.log 2>&1; echo ncu_rc=$?
