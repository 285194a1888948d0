# scene-batch ring sweep (chunk / stages / CTAs per SM); libraries built under exp/ by hand
for i in 1 2; do
for lib in exp/libvfpi_c8s2m3.so exp/libvfpi_c8s3m3.so exp/libvfpi_c4s3m4.so exp/libvfpi_c8s2m4.so exp/libvfpi_c6s2m3.so; do
  echo "== $lib $(VFPI_LIB=$lib timeout 300 python scripts/bench_scenes_kernel.py --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 loop_ms %.2f frac %.3f' % (d['loop_ms'], d['frac']))")"
done; done
