timeout 600 python -m pytest tests/test_gpu_hb2st.py tests/test_gpu_parity.py -x -q -m gpu -k "hb2st" 2>&1 | tail -3
for s in 1; do
  echo "== EIG_HB2ST_SYS=$s"
  EIG_HB2ST_SYS=$s timeout 120 python tools/prof_kernels.py hb2st --n 10000
  EIG_HB2ST_SYS=$s timeout 120 python tools/prof_kernels.py hb2st --n 2000
  EIG_HB2ST_SYS=$s timeout 120 python tools/prof_kernels.py hb2st --n 5000
done
EIG_Q2_PROFILE=1 timeout 120 python tools/prof_kernels.py hb2st --n 10000 2>&1 | tail -1
