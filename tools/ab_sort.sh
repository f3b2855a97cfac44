#!/bin/bash
# A/B of variants/lib_*.so: ncu kernel durations of the tile sorts at config 1 (prof_step) and config 2 (map_step)
mkdir -p gpurun_out
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  for w in "prof_step.py 1" ${AB_MAP-"map_step.py 4"}; do
    SPLAT_B200_LIB=$PWD/$f timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tile_sort -s 6 -c 12 --csv \
      python tools/$w > gpurun_out/abs_${n}_${w%%.*}.csv 2>/dev/null
    python - "$n" "$w" gpurun_out/abs_${n}_${w%%.*}.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[3])) if len(r) > 10]
h = rows[0]; d = {}
for r in rows[1:]:
    k = r[h.index("Kernel Name")].split("(")[0].replace("void ss::", "")
    d.setdefault(k, []).append(float(r[h.index("Metric Value")]))
print(sys.argv[1], sys.argv[2], {k: round(sum(v) / len(v) / 1000, 2) for k, v in d.items()})
PY
  done
done
