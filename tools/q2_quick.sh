timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "q2 or hotpath" 2>&1 | tail -3
for i in 1 2; do python tools/prof_kernels.py q2 --n 10000 --m 10000 --g 32; done
python tools/prof_kernels.py q2 --n 10000 --m 1000 --g 32
python tools/prof_kernels.py q2 --n 2000 --m 2000 --g 32
