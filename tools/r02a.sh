export PYTHONUNBUFFERED=1
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02a_smi.txt
timeout 600 python -m pytest tests -m gpu -x -q > $O/r02a_pytest.log 2>&1; echo pytest=$?
timeout 400 python bench.py > $O/r02a_bench.json 2> $O/r02a_bench.err; echo bench=$?
nproc; lscpu | grep "Model name"
