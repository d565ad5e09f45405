export PYTHONUNBUFFERED=1
O=gpurun_out
export MDG_LIB=tools/variants/libmdg_pen.so
for pen in 1 3 6; do
  export MDG_FALL_PENALTY=$pen
  echo "=== penalty $pen"
  MDG_PLAN_DEBUG=1 python tools/rounds_probe.py 300 200 11 7 2>&1 | grep "fold\] j=. c=[67]\|^c=[67]\|sum round"
  MDG_PLAN_DEBUG=1 python tools/rounds_probe.py 128 64 1 2>&1 | grep "fold\] j=. c=[567]\|^c=[67]\|sum round" | sort -u
  for s in 2 3; do python tools/rounds_probe.py 128 64 $s 2>&1 | grep "sum round"; done
  timeout 300 python bench.py --no-cpu-baseline --no-strong --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench value', d['value'], 'e2e', d['e2e']['value'], 'roofline', d['roofline']['achieved'])"
done > $O/r03j_pen.log 2>&1
