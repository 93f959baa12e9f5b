# 3M short-K engine variant (64 x 32 tiles, 2 CTAs/SM) on vs off: GEMM shapes, he2hb, hot path
for sk in 0 256; do
  echo "== EIG_ZGEMM_SHORTK=$sk"
  export EIG_ZGEMM_SHORTK=$sk
  python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --m3
  python tools/prof_kernels.py gemm --n 4000 --m 4000 --kw 256 --k 4000 --m3
  python tools/prof_kernels.py he2hb --n 10000 --m3
  python tools/prof_kernels.py he2hb --n 2000 --m3
  python bench.py --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['roofline']['stage_tflops'])"
done
