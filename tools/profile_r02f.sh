# r02 final captures: bench launch list, Q2 3M wavefront full, the zgemm variants, panel, systolic hb2st
R=${1:-r02f}
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-zhegv > gpurun_out/plain_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-zhegv > gpurun_out/ncu_launches_$R.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$R.csv > gpurun_out/launches_${R}_summary.txt 2>&1
bash tools/profile_q2_3m.sh $R
python tools/prof_ncu_targets.py $R
for f in gpurun_out/ncu_*_full_${R}_summary.txt; do echo "== $f"; head -8 $f; done
