#!/bin/bash
# registration A/B, alternating: B=1 and B=8 rates of two libraries, three rounds
for r in 1 2 3; do
  for v in "$@"; do
    lib=$PWD/variants/$v.so
    printf "%s " $v; SPLAT_B200_LIB=$lib DEVICE_SCANS=1 python tools/reg_batch_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v['registrations_per_s']) for k,v in d.items() if k in ('1','8','single')})"
  done
done
