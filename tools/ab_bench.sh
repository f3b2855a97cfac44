#!/bin/bash
# Run bench.py once per variants/lib_*.so (A/B), stage times only.
mkdir -p gpurun_out
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  SPLAT_B200_LIB=$PWD/$f timeout 300 python bench.py --steps ${1:-20} --no-cpu-baseline --no-secondary > gpurun_out/ab_$n.log 2>&1
  python - "$n" gpurun_out/ab_$n.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    st = d["stage_ms"]
    print(f"{sys.argv[1]:24s} {d['value']:8.1f} r/s  " + " ".join(f"{k}={v*1000:.0f}" for k, v in st.items() if v))
except Exception as e:
    print(sys.argv[1], "FAILED", e, open(sys.argv[2]).read()[-500:])
PY
done
