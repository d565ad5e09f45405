# Round-end bench lines and the configs report (one B200, through gpurun)
export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 400 python bench.py > $O/r01_bench.json 2> $O/r01_bench.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/r01_bench_reference.json 2>&1; echo ref=$?
timeout 900 python tools/configs_report.py --cap4 7 --out $O/r01_configs_report.json > $O/configs.log 2>&1; echo configs=$?
