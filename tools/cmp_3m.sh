# 4M vs 3M complex GEMM engine: square / he2hb / back-transform shapes, he2hb, hot path
for m3 in "" "--m3"; do
  echo "== m3=$m3"
  python tools/prof_kernels.py gemm --n 8192 $m3
  python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 $m3
  python tools/prof_kernels.py he2hb --n 10000 $m3
  python tools/prof_kernels.py he2hb --n 2000 $m3
done
