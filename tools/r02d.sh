# GPU tests (group split path, witness plan tag, hist rewrite), hist timing, full bench
export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/r02d_pytest.log 2>&1; echo pytest=$?
python tools/hist_target.py --c 5 --reps 5 > $O/r02d_hist.log 2>&1; echo hist=$?
timeout 600 python bench.py > $O/r02d_bench.json 2> $O/r02d_bench.err; echo bench=$?
