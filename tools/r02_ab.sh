#!/bin/bash
# A/B of library variants on the config-1 step: stage times (bench --no-secondary)
mkdir -p gpurun_out
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu-baseline > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(f'{sys.argv[1]:14s} ms/step {d["ms_per_step"]:.4f}', {k: round(v * 1e3, 1) for k, v in d["stage_ms"].items() if v})
PY
}
for spec in "$@"; do
  IFS=: read name envs <<< "$spec"
  run $name $envs
done
