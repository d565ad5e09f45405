export PYTHONUNBUFFERED=1
O=gpurun_out
for s in 3 4 5 6; do
  timeout 600 python bench.py --streams $s --no-cpu-baseline --no-strong --no-configs > $O/r02ab_bench_s$s.json 2>/dev/null; echo s$s=$?
done
timeout 900 python -m pytest tests -m gpu -x -q -k "stress" > $O/r02ab_stress.log 2>&1; echo stress=$?
