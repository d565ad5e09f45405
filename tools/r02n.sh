export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 0 --cutoff 24 --reps 2 > $O/r02n_c7j0.log 2>&1
python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 1 --cutoff 23 --reps 2 > $O/r02n_c7j1.log 2>&1
for i in 1 2; do python tools/ncu_target.py --n 256 --k 32 --seed 7 --c 9 --j 0 --cutoff 77 --reps 3 >> $O/r02n_cfg3_c9.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline > $O/r02n_bench.json 2> $O/r02n_bench.err; echo bench=$?
timeout 600 python bench.py --no-cpu-baseline --no-strong > $O/r02n_bench2.json 2> $O/r02n_bench2.err; echo bench2=$?
