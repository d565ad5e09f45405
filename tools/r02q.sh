export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/batch_timing.py host > $O/r02q_batch_timing.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-strong --no-configs > $O/r02q_bench.json 2> $O/r02q_bench.err; echo bench=$?
timeout 600 python bench.py --no-cpu-baseline --no-strong --no-configs > $O/r02q_bench2.json 2> $O/r02q_bench2.err; echo bench=$?
timeout 1500 python -m pytest tests -m gpu -x -q -k "gamma or permutation or min_weight or golden or cfg" > $O/r02q_pytest.log 2>&1; echo pytest=$?
