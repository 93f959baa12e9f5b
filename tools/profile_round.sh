#!/bin/bash
# Round profiling recipe (B200_PROFILING.md): plain run, launch list, full capture of the top kernels.
set -x
R=${1:-r01}
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launches_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:apply_q2 -c 1 -o gpurun_out/q2_full_$R \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_q2_$R.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 600 -c 3 -o gpurun_out/zgemm_full_$R \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_zgemm_$R.log 2>&1
ls -la gpurun_out/
