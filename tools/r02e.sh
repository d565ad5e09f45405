# diagnostics: tile / fold plans and timings of the histogram and config-4 level-7 rounds; ncu captures
export PYTHONUNBUFFERED=1
O=gpurun_out; T=/tmp/prof; mkdir -p $T
MDG_PLAN_DEBUG=1 python tools/hist_target.py --c 5 --reps 3 > $O/r02e_hist_plan.log 2>&1
for j in 0 1; do
  MDG_PLAN_DEBUG=1 python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j $j --cutoff 24 --reps 2 > $O/r02e_cfg4_c7_j$j.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_hist -s 1 -c 1 -o $T/hist -f python tools/hist_target.py --c 5 --reps 2 > $O/r02e_ncu_hist.log 2>&1; echo ncu_hist=$?
ncu -i $T/hist.ncu-rep --page raw --csv > $O/r02e_hist_raw.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tab_round -s 1 -c 1 -o $T/c7j1 -f python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 1 --cutoff 24 --reps 2 > $O/r02e_ncu_c7j1.log 2>&1; echo ncu_c7j1=$?
ncu -i $T/c7j1.ncu-rep --page raw --csv > $O/r02e_c7j1_raw.csv 2>/dev/null
ncu -i $T/c7j1.ncu-rep --page source --csv > $O/r02e_c7j1_source.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tab_round -s 1 -c 1 -o $T/c7j0 -f python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 0 --cutoff 24 --reps 2 > $O/r02e_ncu_c7j0.log 2>&1; echo ncu_c7j0=$?
ncu -i $T/c7j0.ncu-rep --page raw --csv > $O/r02e_c7j0_raw.csv 2>/dev/null
