# SELL ring (scene batches only): full GPU suite, then configs[3] / configs[2] / configs[4] timings
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
lib=paper_2201_09212_b200/libvfpi.so
VFPI_LIB=$lib timeout 300 python scripts/bench_cfg3.py --max-iters 100 --cpu-iters 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print('cfg3 cheb', v['chebyshev'], 'loop_ms %.2f frac %.3f ctas %d' % (v['loop_ms'], v['frac'], v['ctas'])) for v in d['variants']]"
VFPI_LIB=$lib timeout 300 python scripts/bench_scenes_kernel.py --reps 3 2>&1 | tail -1
timeout 600 python scripts/bench_scenes.py > gpurun_out/cfg2_full.json 2> gpurun_out/cfg2_full.err; tail -c 1500 gpurun_out/cfg2_full.json
