#!/bin/bash
# Round profiling recipe (B200_PROFILING.md): plain run, launch list, full captures of the top kernels.
#   bash tools/profile_round.sh r02
set -x
R=${1:-r02}
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-zhegv > gpurun_out/plain_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-zhegv > gpurun_out/ncu_launches_$R.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$R.csv > gpurun_out/launches_${R}_summary.txt 2>&1
# dominant kernel (Q2 wavefront) at the bench size
ncu --set full --clock-control none --import-source on -k regex:apply_q2wave -c 1 -o gpurun_out/q2_full_$R \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-zhegv > gpurun_out/ncu_q2_$R.log 2>&1
python tools/ncu_summary.py gpurun_out/q2_full_$R.ncu-rep > gpurun_out/ncu_q2wave_full_${R}_summary.txt 2>&1
# the two heaviest zgemm instantiations of the step at full size (Q1 / trsm shapes), he2hb's panel and hb2st
python tools/prof_ncu_targets.py $R
ls -la gpurun_out/
