# GPU tests (shared bound, batch prefetch), hist ncu (final), bench, batch timing
export PYTHONUNBUFFERED=1
O=gpurun_out; T=/tmp/prof; mkdir -p $T
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r02j_pytest.log 2>&1; echo pytest=$?
python tools/batch_timing.py host > $O/r02j_batch.log 2>&1
timeout 600 python bench.py > $O/r02j_bench.json 2> $O/r02j_bench.err; echo bench=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_hist -s 1 -c 1 -o $T/hist -f python tools/hist_target.py --c 5 --reps 2 > $O/r02j_ncu_hist.log 2>&1; echo ncu_hist=$?
ncu -i $T/hist.ncu-rep --page raw --csv > $O/r02j_hist_raw.csv 2>/dev/null
ncu -i $T/hist.ncu-rep --page source --csv > $O/r02j_hist_source.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tab_round -s 1 -c 1 -o $T/c7j1 -f python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 1 --cutoff 23 --reps 2 > $O/r02j_ncu_c7j1.log 2>&1; echo ncu_c7j1=$?
ncu -i $T/c7j1.ncu-rep --page raw --csv > $O/r02j_c7j1_raw.csv 2>/dev/null
ncu -i $T/c7j1.ncu-rep --page source --csv > $O/r02j_c7j1_source.csv 2>/dev/null
