# e2e A/B: side-stream upload overlap vs the previous library
for i in 1 2; do
for lib in exp/libvfpi_nooverlap.so paper_2201_09212_b200/libvfpi.so; do
  echo "== $lib"; VFPI_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value %.4g e2e %.4g' % (d['value'], d['e2e']['value']))"
done; done
