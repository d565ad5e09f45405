#!/bin/bash
# tile-plan sweep over tools/sweep.py's rounds (development tool)
for mtx in 16 32 64; do for tpb in 2 4 8; do
  r=$(MDG_MIN_TX=$mtx MDG_TILES_PER_BLOCK=$tpb python tools/sweep.py 2>/dev/null | tail -1)
  echo "mtx=$mtx tpb=$tpb $r"
done; done
