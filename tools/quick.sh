#!/bin/bash
# GPU parity tests + a short bench line (stage times) of the in-tree library.
python -m pytest tests -x -q -m gpu 2>&1 | tail -1
python bench.py --steps 20 --no-cpu-baseline --no-secondary | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(round(d['value'],1), 'r/s e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],3), ' '.join(f'{k}={v*1000:.1f}' for k,v in d['stage_ms'].items() if v))"
