#!/bin/bash
# registration batches: async per-frame chains (default) vs the phased schedule
python -m pytest tests/test_gpu_registration.py -q -m gpu -p no:cacheprovider -x -k "batch" 2>&1 | tail -2
for mode in devcount phased; do
  if [ $mode = phased ]; then export SS_BATCH_PHASED=1; else unset SS_BATCH_PHASED; fi
  echo "== $mode"; DEVICE_SCANS=1 timeout 300 python tools/reg_batch_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['registrations_per_s']) for k,v in d.items()})"
  SS_BATCH_TIMING=1 python tools/reg_batch_phases.py 2>&1 | tail -2
done
