# hist rewrite timing; stage-1 fold A/B on config 4's level-7 rounds; GPU tests
export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/hist_target.py --c 5 --reps 5 > $O/r02f_hist.log 2>&1; echo hist=$?
for f in default 129 33; do
  for j in 1; do
    if [ $f = default ]; then unset MDG_FORCE_FOLD; else export MDG_FORCE_FOLD=$f; fi
    python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j $j --cutoff 23 --reps 2 > $O/r02f_fold_${f}_j$j.log 2>&1
  done
done
unset MDG_FORCE_FOLD
for f in default 17 34; do
  if [ $f = default ]; then unset MDG_FORCE_FOLD; else export MDG_FORCE_FOLD=$f; fi
  python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 7 --j 0 --cutoff 24 --reps 2 > $O/r02f_fold_${f}_j0.log 2>&1
done
unset MDG_FORCE_FOLD
timeout 1500 python -m pytest tests -m gpu -x -q -k "not sanitizer" > $O/r02f_pytest.log 2>&1; echo pytest=$?
timeout 1500 python -m pytest tests -m gpu -x -q -k "sanitizer" > $O/r02f_sanitizer.log 2>&1; echo sanitizer=$?
