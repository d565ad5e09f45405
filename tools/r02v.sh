# round-2 measurements: full bench (both arms), launch list of the bench, configs report
export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 900 python bench.py > $O/r02v_bench.json 2> $O/r02v_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r02v_bench_reference.json 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02v_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong --no-configs --streams 1 > $O/r02v_ncu3.log 2>&1; echo ncu3=$?
timeout 1800 python tools/configs_report.py --cap4 7 --out $O/r02v_configs_report.json > $O/r02v_configs.log 2>&1; echo configs=$?
