# hb2st n = 10^4: five fresh processes (spread of the position-stationary kernel)
for r in 1 2 3 4 5; do timeout 120 python tools/prof_kernels.py hb2st --n 10000 | tail -1; done
