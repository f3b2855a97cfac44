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
  python tools/sass_regions.py gpurun_out/prof_round.ncu-rep "^k_forward$"
} > profiles/${tag}_ncu_full_summary.txt
cat profiles/${tag}_ncu_full_summary.txt | head -12
if [ -f gpurun_out/prof_map.ncu-rep ]; then
  {
    echo "# ncu --set full (clock-control none), config-2 mapping refine (tools/map_step.py), B200"
    python tools/ncu_summary.py gpurun_out/prof_map.ncu-rep
    echo
    echo "# SASS regions of k_forward_long"
    python tools/sass_regions.py gpurun_out/prof_map.ncu-rep k_forward_long
  } > profiles/${tag}_ncu_map_summary.txt
fi
if [ -f gpurun_out/prof_reg.ncu-rep ]; then
  {
    echo "# ncu --set full (clock-control none), config-3 geometric registration (tools/geo_probe.py), B200"
    python tools/ncu_summary.py gpurun_out/prof_reg.ncu-rep
    echo
    echo "# SASS regions of k_reg_solve"
    python tools/sass_regions.py gpurun_out/prof_reg.ncu-rep k_reg_solve 0.01
  } > profiles/${tag}_ncu_reg_summary.txt
fi
# per-launch DRAM bytes of the config-1 kernels, read by bench.py's roofline.traffic
ncu -i gpurun_out/prof_round.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,json,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; out={'source': 'ncu --set full --clock-control none, tools/prof_step.py config 1, profiles/${tag}_ncu_full_summary.txt (bytes per launch)'}
for r in rows[2:]:
  d=dict(zip(h,r)); sc={'Mbyte':1e6,'Kbyte':1e3,'Gbyte':1e9,'byte':1}
  f=lambda k: float(d[k].replace(',',''))*sc[rows[1][h.index(k)]]
  name=d['Kernel Name'].split('(')[0].replace('void ','')
  key=name.split('<')[0]+('<8>' if name.startswith(('k_forward<','k_backward<')) else '')
  out.setdefault(key, int(round(f('dram__bytes_read.sum')+f('dram__bytes_write.sum'))))
json.dump(out, open('profiles/r02_traffic.json','w')); print(out)
"
python tools/ncu_pipes.py gpurun_out/prof_round.ncu-rep >> profiles/${tag}_ncu_full_summary.txt
