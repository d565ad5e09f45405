# hist: tile plan sweep (suffix size, per-tile overhead) at config 5 level 5
export PYTHONUNBUFFERED=1
O=gpurun_out
for s in default 2 3 4; do
  if [ $s = default ]; then unset MDG_FORCE_S; else export MDG_FORCE_S=$s; fi
  for ov in default 16 64; do
    if [ $ov = default ]; then unset MDG_TILE_OVERHEAD; else export MDG_TILE_OVERHEAD=$ov; fi
    echo "== s=$s overhead=$ov" >> $O/r02i_hist_sweep.log
    MDG_PLAN_DEBUG=1 python tools/hist_target.py --c 5 --reps 3 >> $O/r02i_hist_sweep.log 2>&1
  done
done
unset MDG_FORCE_S MDG_TILE_OVERHEAD
python tools/hist_target.py --c 4 --reps 3 >> $O/r02i_hist_sweep.log 2>&1
