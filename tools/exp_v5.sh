EIG_ZGEMM_V5=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sliced.py -x -q -m gpu 2>&1 | tail -1
for v in 0 1; do
  echo "== EIG_ZGEMM_V5=$v"
  export EIG_ZGEMM_V5=$v
  python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --m3 | tail -4
  python tools/prof_kernels.py he2hb --n 10000 --m3
  python tools/prof_kernels.py he2hb --n 2000 --m3
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-zhegv 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', round(d['value'],3), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['stages_ms'].items()})"
done
