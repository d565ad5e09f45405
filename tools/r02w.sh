# stage-1 choice at config 2's levels 6 and 7 (seed 1, the loop's U): plan vs forced single / pair folds
export PYTHONUNBUFFERED=1
O=gpurun_out
for c in 6 7; do
  if [ $c = 6 ]; then U=16; else U=15; fi
  for f in default 1 65; do
    if [ $f = default ]; then unset MDG_FORCE_FOLD; else export MDG_FORCE_FOLD=$f; fi
    echo "== c=$c fold=$f" >> $O/r02w_fold.log
    python tools/ncu_target.py --c $c --cutoff $U --reps 4 >> $O/r02w_fold.log 2>&1
  done
done
