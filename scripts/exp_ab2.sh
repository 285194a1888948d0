for lib in exp/libvfpi_old.so paper_2201_09212_b200/libvfpi.so exp/libvfpi_old.so paper_2201_09212_b200/libvfpi.so; do
  echo "== $lib"
  VFPI_LIB=$lib timeout 300 python scripts/bench_cfg3.py --max-iters 100 --cpu-iters 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print('cfg3 cheb', v['chebyshev'], 'loop_ms %.2f frac %.3f ctas %d' % (v['loop_ms'], v['frac'], v['ctas'])) for v in d['variants']]"
  VFPI_LIB=$lib timeout 300 python scripts/bench_scenes_kernel.py --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 loop_ms %.2f frac %.3f' % (d['loop_ms'], d['frac']))"
done
VFPI_LIB=exp/libvfpi_old.so timeout 300 python scripts/bench_cfg4.py --steps 56 --max-iters 100 --cpu-iters 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old cfg4 loop_s %.3f frac %.3f' % (d['loop']['loop_s'], d['loop']['frac']))"
timeout 300 python scripts/bench_cfg4.py --steps 56 --max-iters 100 --cpu-iters 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new cfg4 loop_s %.3f frac %.3f' % (d['loop']['loop_s'], d['loop']['frac']))"
