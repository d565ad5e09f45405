#!/bin/bash
# CLI wall time per invocation (CUDA init + module load + run), lazy vs eager module loading
B=paper_1911_08963_b200/bin/mindist
$B gen --n 80 --k 40 --seed 1 > /tmp/c1.txt
$B gen --n 128 --k 64 --seed 1 > /tmp/c2.txt
for mode in LAZY EAGER LAZY EAGER; do
  for f in /tmp/c1.txt /tmp/c2.txt; do
    t=""
    for i in 1 2 3; do
      s=$(date +%s.%N); CUDA_MODULE_LOADING=$mode $B mindist $f --seed 1 > /dev/null 2>&1; e=$(date +%s.%N)
      t="$t $(python3 -c "print(round($e-$s,3))")"
    done
    echo "$mode $f:$t"
  done
done
