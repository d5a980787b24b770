#!/bin/bash
# isolated k_layer_hist launch times (ncu, host masks so nothing overlaps)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_layer_hist --csv python tools/prof_fit.py --trees 8 --reps 1 --host-masks 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; i=h.index('Metric Value'); u=h.index('Metric Unit')
v=[float(r[i].replace(',',''))*(1e-3 if r[u] in ('nsecond','ns') else 1) for r in rows[1:]]
print('hist launches', len(v), 'avg us %.1f' % (sum(v)/len(v)), 'per layer', ['%.1f' % x for x in v[:6]])
"
