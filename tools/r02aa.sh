export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/hist_target.py --c 5 --reps 3 > $O/r02aa_hist.log 2>&1
for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -x -q -k "multi or group" >> $O/r02aa_multi.log 2>&1; echo multi$i=$?; done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r02aa_pytest.log 2>&1; echo pytest=$?
