#!/usr/bin/env python
"""ncu --set full captures of single kernels at full size (n = 10^4), one
process each: the zgemm instantiations that dominate the step, the panel
kernel and the bulge chase.  Writes <name>_<round>.ncu-rep and a summary."""
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
T = [
    # (name, kernel regex, skip count, command); zgemm_kernel<OPA, OPB, HERM, LOWER, variant>
    ("zgemm_CN", "regex:zgemm_kernel<.int.1, .int.0, .bool.0, .int.0, .int.4>", 0,
     "python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --reps 1 --m3"),
    ("zgemm_NN", "regex:zgemm_kernel<.int.0, .int.0, .bool.0, .int.0, .int.4>", 1,
     "python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --reps 1 --m3"),
    ("her2k", "regex:zgemm_kernel<.int.0, .int.1, .bool.0, .int.1, .int.2>", 1,
     "python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --reps 1 --m3"),
    ("hemm", "regex:zgemm_kernel<.int.0, .int.0, .bool.1, .int.0, .int.2>", 1,
     "python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --reps 1 --m3"),
    ("panel", "regex:panel_qr_kernel", 20, "python tools/prof_kernels.py he2hb --n 10000 --reps 1"),
    ("hb2sys", "regex:hb2sys_kernel", 0, "python tools/prof_kernels.py hb2st --n 10000 --reps 1"),
]
for name, k, skip, cmd in T:
    rep = f"gpurun_out/{name}_full_{R}"
    subprocess.run(f"ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k '{k}' -s {skip} -c 1 -o {rep} {cmd} "
                   f"> gpurun_out/ncu_{name}_{R}.log 2>&1", shell=True)
    subprocess.run(f"python tools/ncu_summary.py {rep}.ncu-rep > gpurun_out/ncu_{name}_full_{R}_summary.txt 2>&1",
                   shell=True)
