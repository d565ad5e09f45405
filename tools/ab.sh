#!/bin/bash
# A/B tools/sweep.py's rounds (+ config 4's level-6 rounds) across library builds
for lib in paper_1911_08963_b200/lib/libmdg.so tools/variants/*.so; do
  r=$(MDG_LIB=$lib python tools/sweep.py 2>/dev/null | tail -1)
  a=$(MDG_LIB=$lib python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 6 --j 1 --cutoff 24 --reps 2 2>&1 | tail -1 | grep -o "ms=[0-9.]*")
  b=$(MDG_LIB=$lib python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 6 --j 0 --cutoff 24 --reps 2 2>&1 | tail -1 | grep -o "ms=[0-9.]*")
  echo "$(basename $lib) $r c6j1 $a c6j0 $b"
done
