#!/bin/bash
# isolated layer-histogram launch times per path (ncu, host masks); extra
# variants via HP_EXTRA="NAME:ENV=VAL ..." (e.g. fl_noflush:BB_FL_NOFLUSH=1)
run() {
  echo "== $1"
  env $2 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_layer_hist --csv \
    python tools/prof_fit.py ${PF_ARGS:---trees 4 --reps 1 --host-masks} 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; i=h.index('Metric Value'); u=h.index('Metric Unit'); k=h.index('Kernel Name')
v=[float(r[i].replace(',',''))*(1e-3 if r[u] in ('nsecond','ns') else 1) for r in rows[1:]]
L=int(__import__('os').environ.get('PF_DEPTH','3')); print('kernel', rows[1][k][:40], 'launches', len(v), 'avg us %.1f' % (sum(v)/len(v)), 'per layer', ['%.1f' % (sum(v[l::L])/len(v[l::L])) for l in range(L)])
"
}
run fl BB_HIST_PATH=fl
run w BB_HIST_PATH=w
for x in $HP_EXTRA; do run "${x%%:*}" "BB_HIST_PATH=fl ${x#*:}"; done
