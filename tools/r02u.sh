export PYTHONUNBUFFERED=1
O=gpurun_out
for v in default hist5 hist6; do
  if [ $v = default ]; then L=paper_1911_08963_b200/lib/libmdg.so; else L=tools/variants/libmdg_$v.so; fi
  echo "== $v" >> $O/r02u_hist.log
  MDG_LIB=$L python tools/hist_target.py --c 5 --reps 4 >> $O/r02u_hist.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r02u_pytest.log 2>&1; echo pytest=$?
