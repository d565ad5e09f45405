export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r02x_pytest.log 2>&1; echo pytest=$?
