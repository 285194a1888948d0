# streaming-kernel variants (exp/libvfpi_*.so): configs[3] solve and configs[2] batch kernel timing
for lib in paper_2201_09212_b200/libvfpi.so exp/libvfpi_v1.so exp/libvfpi_v2.so exp/libvfpi_v3.so exp/libvfpi_v4.so; do
  echo "== $lib"
  VFPI_LIB=$lib timeout 300 python scripts/bench_cfg3.py --max-iters 100 --cpu-iters 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print('cfg3 cheb', v['chebyshev'], 'loop_ms %.2f frac %.3f ctas %d' % (v['loop_ms'], v['frac'], v['ctas'])) for v in d['variants']]"
  VFPI_LIB=$lib timeout 300 python scripts/bench_scenes_kernel.py --reps 3 2>&1 | tail -1
done
