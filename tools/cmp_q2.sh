# Q2 wavefront variants (EIG_LIB) at the bench size and the P = 8 per-rank size; panel CTA cap sweep
for lib in paper_1207_1773_b200/libeigb200.so .cmp/lib_q2s3.so; do
  echo "== $lib"
  for m in 10000 1250 1000; do EIG_LIB=$lib python tools/prof_kernels.py q2 --n 10000 --m $m --g 32 --reps 3; done
done
for c in 8 12 16 24 32; do
  echo "== EIG_PANEL_CTAS=$c"
  for n in 2000 5000; do EIG_PANEL_CTAS=$c python tools/prof_kernels.py he2hb --n $n --reps 3; done
done
