export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not cap7" > $O/r02t_pytest.log 2>&1; echo pytest=$?
python tools/batch_timing.py host > $O/r02t_batch_timing.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-strong --no-configs > $O/r02t_bench.json 2> $O/r02t_bench.err; echo bench=$?
