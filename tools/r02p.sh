export PYTHONUNBUFFERED=1
O=gpurun_out
python tools/batch_timing.py host gpu > $O/r02p_batch_timing.log 2>&1
MDG_HOST_THREADS=8 python tools/batch_timing.py host > $O/r02p_batch_timing_ht8.log 2>&1
MDG_HOST_THREADS=4 python tools/batch_timing.py host > $O/r02p_batch_timing_ht4.log 2>&1
