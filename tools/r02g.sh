# e2e / value vs codes in flight
export PYTHONUNBUFFERED=1
O=gpurun_out
for s in 4 8; do
  timeout 600 python bench.py --streams $s --no-cpu-baseline --no-strong --no-configs > $O/r02g_bench_s$s.json 2> $O/r02g_bench_s$s.err; echo s$s=$?
done
