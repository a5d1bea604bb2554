#!/bin/bash
# SM clock / power while a CG form runs (nvidia-smi every 100 ms).
for f in "two" "pass"; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 > gpurun_out/pw_$f.csv &
  P=$!
  if [ $f = pass ]; then CF_CG_ALGO=pass python tools/probe_cg.py --n 256 --iters 3000 --repeat 3; else python tools/probe_cg.py --n 256 --iters 3000 --repeat 3; fi
  kill $P
  python3 -c "
import statistics as s
rows=[l.strip().split(', ') for l in open('gpurun_out/pw_$f.csv') if l.strip()]
busy=[r for r in rows if float(r[1])>400]
print('$f', 'samples',len(busy),'sm_mhz median',s.median(float(r[0]) for r in busy),'power median',s.median(float(r[1]) for r in busy), 'capped', sum(1 for r in busy if 'Active' in r[2]))
"
done
