#!/bin/bash
# tile-plan sweep over tools/sweep.py's rounds (development tool)
for ov in 0 4 8; do for tpb in 2 4 8; do
  r=$(MDG_TILE_OVERHEAD=$ov MDG_TILES_PER_BLOCK=$tpb python tools/sweep.py 2>/dev/null | tail -1)
  echo "ov=$ov tpb=$tpb $r"
done; done
