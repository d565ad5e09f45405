# GPU tests of the new build, histogram timing + ncu of tab_hist (cfg5 c=5)
export PYTHONUNBUFFERED=1
O=gpurun_out; T=/tmp/prof; mkdir -p $T
timeout 900 python -m pytest tests -m gpu -x -q > $O/r02b_pytest.log 2>&1; echo pytest=$?
python tools/hist_target.py --c 5 --reps 5 > $O/r02b_hist.log 2>&1; echo hist=$?
python tools/hist_target.py --c 4 --reps 3 >> $O/r02b_hist.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_hist -s 1 -c 1 -o $T/hist -f python tools/hist_target.py --c 5 --reps 2 > $O/r02b_ncu.log 2>&1; echo ncu=$?
ncu -i $T/hist.ncu-rep --page raw --csv > $O/r02b_hist_raw.csv 2>/dev/null
ncu -i $T/hist.ncu-rep --page details > $O/r02b_hist_details.txt 2>/dev/null
ncu -i $T/hist.ncu-rep --page source --csv > $O/r02b_hist_source.csv 2>/dev/null
