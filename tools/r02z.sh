export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r02z_pytest.log 2>&1; echo pytest=$?
python tools/hist_target.py --c 5 --reps 3 > $O/r02z_hist.log 2>&1
