# ncu captures: config 3 level-9 round (NW 7, m = 8), its fused levels, and the rd kernel on config 2 level 7
export PYTHONUNBUFFERED=1
O=gpurun_out; T=/tmp/prof; mkdir -p $T
python tools/rounds_probe.py 256 32 7 > $O/r02r_cfg3_rounds.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_round -s 2 -c 1 -o $T/cfg3 -f python tools/ncu_target.py --n 256 --k 32 --seed 7 --c 9 --j 0 --cutoff 77 --reps 3 > $O/r02r_ncu_cfg3.log 2>&1; echo ncu_cfg3=$?
ncu -i $T/cfg3.ncu-rep --page raw --csv > $O/r02r_cfg3_raw.csv 2>/dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_round -s 2 -c 1 -o $T/rd -f python tools/ncu_target.py --kernel rd --cutoff 16 --reps 3 > $O/r02r_ncu_rd.log 2>&1; echo ncu_rd=$?
ncu -i $T/rd.ncu-rep --page raw --csv > $O/r02r_rd_raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02r_launches_cfg3.csv python tools/rounds_probe.py 256 32 7 > $O/r02r_ncu_cfg3_launches.log 2>&1; echo ncu_l=$?
