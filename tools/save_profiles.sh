#!/bin/bash
# Copy the evidence of the last round_profile.sh call into profiles/ under tag $1 (e.g. r01_v4).
set -e
cd "$(dirname "$0")/.."
tag=$1
tail -1 gpurun_out/bench.log > profiles/${tag}_bench.json
cp gpurun_out/launches.csv profiles/${tag}_bench_launches.csv
{
  echo "# ncu --set full (clock-control none), config-1 step loop (tools/prof_step.py), one launch per kernel, B200"
  python tools/ncu_summary.py gpurun_out/prof_round.ncu-rep
  echo
  echo "# DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)"
  ncu -i gpurun_out/prof_round.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[2:]:
  d=dict(zip(h,r)); f=lambda k: float(d[k].replace(',',''))
  print(d['Kernel Name'].split('(')[0], 'read', f('dram__bytes_read.sum'), 'write', f('dram__bytes_write.sum'), d['dram__bytes_read.sum'] and '')
"
  echo
  echo "# SASS regions of k_backward (runs of equal execution count)"
  python tools/sass_regions.py gpurun_out/prof_round.ncu-rep k_backward
  echo
  echo "# SASS regions of k_forward"
  python tools/sass_regions.py gpurun_out/prof_round.ncu-rep k_forward
} > profiles/${tag}_ncu_full_summary.txt
cat profiles/${tag}_ncu_full_summary.txt | head -12
