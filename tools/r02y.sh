export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/hist_target.py --c 5 --reps 5 > $O/r02y_hist.log 2>&1; echo hist=$?
python tools/hist_target.py --c 4 --reps 3 >> $O/r02y_hist.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "hist or smoke" > $O/r02y_pytest.log 2>&1; echo pytest=$?
