export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/e2e_probe.py > $O/r02o_e2e_probe.log 2>&1
MDG_TIMING=1 MDG_PLAN_DEBUG=1 python tools/front_once.py > $O/r02o_front_once.log 2>&1
MDG_TIMING=1 python tools/batch_timing.py host > $O/r02o_batch_timing.log 2>&1
