# Q2 wavefront variants (EIG_LIB) at the bench size and the P = 8 per-rank size
for lib in paper_1207_1773_b200/libeigb200.so .cmp/lib_q2w13.so .cmp/lib_q2w14.so; do
  echo "== $lib"
  for m in 10000 1250; do EIG_LIB=$lib python tools/prof_kernels.py q2 --n 10000 --m $m --g 32 --reps 3; done
done
