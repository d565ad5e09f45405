# Round-end measurements on one B200 (run through gpurun): bench (both arms), ncu --set full
# of the level-7 round and of the fused level-7 launch (summaries + raw CSV pages), launch list
export PYTHONUNBUFFERED=1
O=gpurun_out; T=/tmp/prof; mkdir -p $T
timeout 400 python bench.py > $O/r01m_bench.json 2> $O/r01m_bench.err; echo bench=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_round -s 2 -c 1 -o $T/c7 -f python tools/ncu_target.py --cutoff 16 --reps 3 > $O/ncu1.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_level -s 13 -c 1 -o $T/level7 -f python tools/rounds_probe.py 128 64 1 > $O/ncu2.log 2>&1; echo ncu2=$?
for r in c7 level7; do
  ncu -i $T/$r.ncu-rep --page raw --csv > $O/r01m_${r}_raw.csv 2>/dev/null
  ncu -i $T/$r.ncu-rep --page source --csv > $O/r01m_${r}_source.csv 2>/dev/null
  ncu -i $T/$r.ncu-rep --page details > $O/r01m_${r}_details.txt 2>/dev/null
done
ls -la $T
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r01m_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 > $O/ncu3.log 2>&1; echo ncu3=$?
du -sh $O/*
