# Q2 wavefront: 3M form (default) vs real embedding (EIG_Q2_3M=0)
for q in 0 1; do
  echo "== EIG_Q2_3M=$q"
  export EIG_Q2_3M=$q
  python tools/prof_kernels.py q2 --n 10000 --m 10000 --g 32
  python tools/prof_kernels.py q2 --n 10000 --m 1000 --g 32
  python tools/prof_kernels.py q2 --n 2000 --m 2000 --g 32
  python bench.py --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['roofline']['stage_tflops'])"
done
