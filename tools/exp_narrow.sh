./tools/peaks/dmma_dadd
for nw in 0 64; do
  echo "== NARROW=$nw"
  export EIG_ZGEMM_NARROW=$nw
  python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --m3 | grep hemm
  python tools/prof_kernels.py gemm --n 2000 --m 2000 --kw 256 --k 2000 --m3 | grep hemm
  python tools/prof_kernels.py he2hb --n 10000 --m3
  python tools/prof_kernels.py he2hb --n 2000 --m3
done
