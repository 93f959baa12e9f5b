# A/B of two builds of libeigb200 (EIG_LIB): he2hb / hb2st timings and panel phases
for lib in .cmp/libeig_old.so paper_1207_1773_b200/libeigb200.so; do
  echo "== $lib"
  for n in 10000 2000; do EIG_LIB=$lib python tools/prof_kernels.py he2hb --n $n --reps 3; done
  EIG_LIB=$lib EIG_Q2_PROFILE=1 python tools/prof_kernels.py he2hb --n 10000 --reps 1
  EIG_LIB=$lib python tools/prof_kernels.py hb2st --n 10000 --reps 3
done
