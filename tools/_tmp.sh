export PYTHONUNBUFFERED=1
O=gpurun_out
timeout 900 python tools/_repro.py 65 620 108 > $O/r03v_repro.log 2>&1; echo repro=$?
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r03v_pytest.log 2>&1; echo pytest=$?
: > $O/r03v_sweep.log
i=0
for code in 0 1 2 4 17 18 33 65 97 129 49; do
  i=$((i+1))
  timeout 900 python tools/forced_sweep.py $code 800 $((100+i)) >> $O/r03v_sweep.log 2>&1
  echo "code $code rc=$?" >> $O/r03v_sweep.log
done
