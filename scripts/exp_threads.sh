for lib in paper_2201_09212_b200/libvfpi.so exp/libvfpi_t384.so exp/libvfpi_t768.so exp/libvfpi_t1024.so; do
  echo "== $lib"; VFPI_LIB=$lib timeout 200 python scripts/exp_bar.py 0 0 2>&1 | tail -1
done
