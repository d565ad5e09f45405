#!/bin/bash
# tile-geometry sweep on the level-7 config-2 round (development tool)
for tpb in 8 16 32 64; do for mtx in 8 16 32; do
  r=$(MDG_TILES_PER_BLOCK=$tpb MDG_MIN_TX=$mtx python tools/ncu_target.py --cutoff 15 --reps 5 2>&1 | tail -1)
  echo "tpb=$tpb min_tx=$mtx $r"
done; done
