import subprocess
R = "r02x"
T = [("zgemm_CN", "regex:zgemm_kernel<.int.1, .int.0, .bool.0, .int.0, .int.4>", 0),
     ("zgemm_NN", "regex:zgemm_kernel<.int.0, .int.0, .bool.0, .int.0, .int.4>", 1)]
cmd = "python tools/prof_kernels.py gemm --n 10000 --m 10000 --kw 256 --k 10000 --reps 1 --m3"
for name, k, skip in T:
    rep = f"gpurun_out/{name}_full_{R}"
    subprocess.run(f"ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k '{k}' -s {skip} -c 1 -o {rep} {cmd} > gpurun_out/ncu_{name}_{R}.log 2>&1", shell=True)
    subprocess.run(f"python tools/ncu_summary.py {rep}.ncu-rep > gpurun_out/ncu_{name}_full_{R}_summary.txt 2>&1", shell=True)
