# A/B of hb2st build variants in .cmp/ (timing only)
for v in "$@"; do echo "== $v"; EIG_LIB=.cmp/lib_hb_$v.so timeout 120 python tools/prof_kernels.py hb2st --n 10000 2>&1 | tail -1; done
