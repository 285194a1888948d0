for lib in exp/libvfpi_u8.so exp/libvfpi_u4.so exp/libvfpi_u6.so exp/libvfpi_u12.so exp/libvfpi_u16.so; do
  echo "== $lib"
  VFPI_LIB=$lib timeout 300 python scripts/bench_cfg3.py --max-iters 100 --cpu-iters 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print('cfg3 cheb', v['chebyshev'], 'loop_ms %.2f frac %.3f ctas %d' % (v['loop_ms'], v['frac'], v['ctas'])) for v in d['variants']]"
  VFPI_LIB=$lib timeout 300 python scripts/bench_cfg4.py --steps 56 --max-iters 100 --cpu-iters 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 loop_s %.3f frac %.3f' % (d['loop']['loop_s'], d['loop']['frac']))"
  VFPI_LIB=$lib timeout 300 python scripts/bench_scenes_kernel.py --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 loop_ms %.2f frac %.3f' % (d['loop_ms'], d['frac']))"
done
