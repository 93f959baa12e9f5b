# ncu --set full of the 3M Q2 wavefront (bench size), plus its source page
R=${1:-r02c}
ncu --set full --clock-control none --import-source on -k regex:apply_q2wave -c 1 -o gpurun_out/q2_full_$R \
    python tools/prof_kernels.py q2 --n 10000 --g 32 --reps 1 > gpurun_out/ncu_q2_$R.log 2>&1
python tools/ncu_summary.py gpurun_out/q2_full_$R.ncu-rep > gpurun_out/ncu_q2wave_full_${R}_summary.txt 2>&1
ncu -i gpurun_out/q2_full_$R.ncu-rep --page source --csv --print-source sass > gpurun_out/q2_src_$R.csv 2>/dev/null
head -40 gpurun_out/ncu_q2wave_full_${R}_summary.txt
