# quick status: Q2 small m (per-rank load at P = 8), he2hb n = 2000, hb2st n = 10^4
python tools/prof_kernels.py q2 --n 10000 --m 1250 --g 32
python tools/prof_kernels.py q2 --n 10000 --m 1000 --g 32
python tools/prof_kernels.py he2hb --n 2000 --m3
python tools/prof_kernels.py he2hb --n 5000 --m3
python tools/prof_kernels.py hb2st --n 10000
python tools/prof_kernels.py hb2st --n 2000
