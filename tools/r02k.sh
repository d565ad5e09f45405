# e2e vs Gamma searches ahead of the loops
export PYTHONUNBUFFERED=1
O=gpurun_out
for a in 0 1 2 4; do
  MDG_GAMMA_AHEAD=$a python tools/batch_timing.py host > $O/r02k_batch_a$a.log 2>&1
  MDG_GAMMA_AHEAD=$a timeout 600 python bench.py --no-cpu-baseline --no-strong --no-configs > $O/r02k_bench_a$a.json 2>/dev/null; echo a$a=$?
done
