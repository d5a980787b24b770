#!/bin/bash
# knob sweep for the cfg2 fit (device-timed value only)
run() { env "$@" timeout 120 python bench.py --steps 5 --no-e2e --no-cpu --no-apply 2>/dev/null | tail -1 | python -c "import sys,json;d=json.loads(sys.stdin.read());print('$*', round(d['value']/1e9,4), round(d['ms_per_step'],2))"; }
for rep in 1 2; do
  run BB_X=0
  for sd in 1.0 1.5 3.0; do run BB_ANCHOR_SD=$sd; done
  for r in 0 4 14; do run BB_HIST_RESERVE=$r; done
  for p in 1 2; do run BB_MASK_PRIO=$p; done
done
