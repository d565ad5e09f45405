# hist (xi unroll) timing + ncu; pipe microbenchmark with the per-SM clock fix
export PYTHONUNBUFFERED=1
O=gpurun_out; T=/tmp/prof; mkdir -p $T
python tools/hist_target.py --c 5 --reps 5 > $O/r02h_hist.log 2>&1; echo hist=$?
./tools/pipes_microbench > $O/r02h_pipes_microbench.jsonl 2>&1; echo pipes=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_hist -s 1 -c 1 -o $T/hist -f python tools/hist_target.py --c 5 --reps 2 > $O/r02h_ncu_hist.log 2>&1; echo ncu_hist=$?
ncu -i $T/hist.ncu-rep --page raw --csv > $O/r02h_hist_raw.csv 2>/dev/null
ncu -i $T/hist.ncu-rep --page source --csv > $O/r02h_hist_source.csv 2>/dev/null
