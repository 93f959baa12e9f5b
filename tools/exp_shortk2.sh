for sk in 256 128; do
  echo "== EIG_ZGEMM_SHORTK=$sk"
  export EIG_ZGEMM_SHORTK=$sk
  python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --m3 | tail -1
  python tools/prof_kernels.py gemm --n 4000 --m 4000 --kw 256 --k 4000 --m3 | tail -1
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-zhegv 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', round(d['value'],3), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stages_ms'].items()})"
done
