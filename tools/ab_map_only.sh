#!/bin/bash
# Config-2 (mapping) stage times of variants/lib_*.so (no parity run).
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  echo "== $n: $(SPLAT_B200_LIB=$PWD/$f timeout 300 python tools/map_stages.py 2>&1 | grep -E 'stages|x200' | tr '\n' ' ')"
done
