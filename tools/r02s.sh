export PYTHONUNBUFFERED=1
O=gpurun_out
for s in default 2; do
  if [ $s = default ]; then unset MDG_FORCE_S; else export MDG_FORCE_S=$s; fi
  for t in 1 2 4 8; do
    echo "== s=$s tpb=$t" >> $O/r02s_hist.log
    MDG_HIST_TPB=$t MDG_PLAN_DEBUG=1 python tools/hist_target.py --c 5 --reps 3 2>&1 | grep -E "c=5|rep 2" >> $O/r02s_hist.log
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "not cap7" > $O/r02s_pytest.log 2>&1; echo pytest=$?
