# Q1 aggregation width (EIG_Q1_KW) at the bench size: stage times of the hot path
for kw in 256 384 512; do
  echo "== EIG_Q1_KW=$kw"
  EIG_Q1_KW=$kw python bench.py --steps 2 --warmup 2 --no-cpu --no-e2e --no-zhegv | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['stages_ms'])"
done
