timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "q2 or hotpath" 2>&1 | tail -3
timeout 120 python tools/prof_kernels.py q2 --n 10000 --m 10000 --g 32
timeout 120 python tools/prof_kernels.py q2 --n 10000 --m 10000 --g 32
timeout 60 python tools/prof_kernels.py q2 --n 10000 --m 1250 --g 32
timeout 60 python tools/prof_kernels.py q2 --n 10000 --m 1000 --g 32
timeout 60 python tools/prof_kernels.py q2 --n 2000 --m 2000 --g 32
