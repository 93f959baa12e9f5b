# Q2 wavefront A/B (EIG_LIB) at the bench size, alternating builds
for r in 1 2; do
for lib in paper_1207_1773_b200/libeigb200.so .cmp/lib_head.so; do
  echo "== $lib"; EIG_LIB=$lib python tools/prof_kernels.py q2 --n 10000 --m 10000 --g 32 --reps 3
done; done
