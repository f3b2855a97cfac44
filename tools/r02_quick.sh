#!/bin/bash
# parity subset + a quick config-1 bench (stage times)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "parity or golden or spec or mapping" > gpurun_out/pytest_quick.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-secondary --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"], 1))
print({k: round(v * 1e3, 1) for k, v in d["stage_ms"].items()})
print("roofline", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), "step", round(d["roofline"]["step_frac"], 3))
PY
