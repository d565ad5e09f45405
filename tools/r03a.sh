# unit-column elision: cfg4 cap-7 per-round times with and without, then the GPU suite
export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/rounds_probe.py 300 200 11 7 > $O/r03a_rounds_on.log 2>&1
MDG_NO_UNIT_ELISION=1 python tools/rounds_probe.py 300 200 11 7 > $O/r03a_rounds_off.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r03a_pytest.log 2>&1; echo pytest=$?
