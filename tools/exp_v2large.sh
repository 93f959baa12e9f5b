for sk in 256 100000000; do
  echo "== EIG_ZGEMM_SHORTK=$sk"
  EIG_ZGEMM_SHORTK=$sk python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --m3
done
