# Final-round captures: launch list of one bench step, the 12-warp Q2 wavefront at the bench size
R=${1:-r02b}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-zhegv > gpurun_out/ncu_launches_$R.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$R.csv > gpurun_out/launches_${R}_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:apply_q2wave -c 1 -o gpurun_out/q2_full_$R \
    python tools/prof_kernels.py q2 --n 10000 --g 32 --reps 1 > gpurun_out/ncu_q2_$R.log 2>&1
python tools/ncu_summary.py gpurun_out/q2_full_$R.ncu-rep > gpurun_out/ncu_q2wave_full_${R}_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:hb2st_kernel -c 1 -o gpurun_out/hb2st_full_$R \
    python tools/prof_kernels.py hb2st --n 10000 --reps 1 > gpurun_out/ncu_hb2st_$R.log 2>&1
python tools/ncu_summary.py gpurun_out/hb2st_full_$R.ncu-rep > gpurun_out/ncu_hb2st_full_${R}_summary.txt 2>&1
cat gpurun_out/launches_${R}_summary.txt; head -14 gpurun_out/ncu_q2wave_full_${R}_summary.txt; head -5 gpurun_out/ncu_hb2st_full_${R}_summary.txt
