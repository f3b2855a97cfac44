#!/bin/bash
# A/B of the batched registration: default library vs variants/rs2.so (2 loop blocks per SM)
mkdir -p gpurun_out
for spec in "main:1:" "rs2:1:variants/rs2.so" "rs2:2:variants/rs2.so"; do
  IFS=: read name bps lib <<< "$spec"
  if [ -n "$lib" ]; then export SPLAT_B200_LIB=$PWD/$lib; else unset SPLAT_B200_LIB; fi
  SS_RS_BPS=$bps DEVICE_SCANS=1 timeout 300 python tools/reg_batch_probe.py > gpurun_out/abreg_${name}_$bps.json 2> gpurun_out/abreg_${name}_$bps.err
  echo "$name bps=$bps: $(python -c "import json;d=json.load(open('gpurun_out/abreg_${name}_$bps.json'));print({k:round(v['registrations_per_s']) for k,v in d.items()})")"
done
