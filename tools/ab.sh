#!/bin/bash
# A/B tools/sweep.py's rounds across library builds (the product lib + tools/variants/*.so)
for lib in paper_1911_08963_b200/lib/libmdg.so tools/variants/*.so; do
  r=$(MDG_LIB=$lib python tools/sweep.py 2>/dev/null | tail -1)
  echo "$(basename $lib) $r"
done
