#!/bin/bash
# A/B the level-7 config-2 round and the config-4 level-5 rounds across library builds
for lib in paper_1911_08963_b200/lib/libmdg.so tools/variants/*.so; do
  a=$(MDG_LIB=$lib python tools/ncu_target.py --cutoff 15 --reps 6 2>&1 | tail -1 | grep -o "cw/s=.*")
  b=$(MDG_LIB=$lib python tools/ncu_target.py --n 300 --k 200 --seed 11 --c 5 --j 0 --cutoff 26 --reps 3 2>&1 | tail -1 | grep -o "cw/s=.*")
  c=$(MDG_LIB=$lib python tools/ncu_target.py --c 6 --cutoff 15 --reps 6 2>&1 | tail -1 | grep -o "cw/s=.*")
  echo "$(basename $lib) cfg2c7 $a | cfg4g0c5 $b | cfg2c6 $c"
done
