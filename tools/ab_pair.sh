# A/B of the stage-1 pair pre-filter (development): config-2 rounds at T = 7, 8, 9, 10,
# the sweep rounds and config 4 level 6, against a baseline library (tools/variants/)
export PYTHONUNBUFFERED=1
for v in "" "MDG_LIB=tools/variants/libmdg_nox2.so"; do
  echo "== $v"
  for cc in "7 15" "7 16" "6 16" "5 16"; do
    set -- $cc
    r=$(env $v python tools/ncu_target.py --c $1 --cutoff $2 --reps 4 2>&1 | tail -1)
    echo "c=$1 cut=$2 $r"
  done
  env $v python tools/sweep.py 2>&1 | tail -1
  env $v python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 6 --j 1 --cutoff 24 --reps 2 2>&1 | tail -1
  env $v python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 6 --j 0 --cutoff 24 --reps 2 2>&1 | tail -1
done
