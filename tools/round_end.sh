# Round-end measurements on one B200 (run through gpurun; outputs under gpurun_out/, the
# summaries worth keeping are copied into profiles/ by hand):
#   GPU suite, bench (both arms), configs report, ncu --set full of the headline level-7 round,
#   of config 4's two level-7 rounds and of the histogram kernel, launch list of the bench.
# Usage: bash tools/round_end.sh TAG   (e.g. r02f)
export PYTHONUNBUFFERED=1
TAG=${1:-rXX}; O=gpurun_out; T=/tmp/prof; mkdir -p $T $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err; echo ref=$?
timeout 900 python tools/configs_report.py --cap4 7 --out $O/${TAG}_configs_report.json > $O/${TAG}_configs.log 2>&1; echo configs=$?
cap() { # cap NAME KERNEL_REGEX SKIP command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 -o $T/$name -f "$@" > $O/${TAG}_ncu_$name.log 2>&1; echo ncu_$name=$?
  ncu -i $T/$name.ncu-rep --page raw --csv > $O/${TAG}_${name}_raw.csv 2>/dev/null
  ncu -i $T/$name.ncu-rep --page source --csv > $O/${TAG}_${name}_source.csv 2>/dev/null
  ncu -i $T/$name.ncu-rep --page details > $O/${TAG}_${name}_details.txt 2>/dev/null
}
cap c7 tab_round 2 python tools/ncu_target.py --cutoff 16 --reps 3
cap cfg4_c7_j0 tab_round 1 python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 0 --cutoff 24 --reps 2
cap cfg4_c7_j1 tab_round 1 python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 1 --cutoff 23 --reps 2
cap hist_c5 tab_hist 1 python tools/hist_target.py --c 5 --reps 2
cap hist_c6 tab_hist 1 python tools/hist_target.py --c 6 --reps 2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong --no-configs --streams 1 > $O/${TAG}_ncu_launches.log 2>&1; echo launches=$?
du -sh $O/${TAG}_* | tail -40
