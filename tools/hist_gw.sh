# per-layer histogram times, global-atomic vs warp kernel vs default (5M-row slices)
for P in g w auto; do
 echo "== $P"
 for CFG in "cfg3 5" "cfg5 6" "cfg2 3"; do set -- $CFG
  BB_HIST_PATH=$P ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_layer_hist --csv python tools/prof_fit.py --config $1 --n 5000000 --trees 2 --reps 1 --host-masks 2>/dev/null | python -c "
import csv,sys
L=$2
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; i=h.index('Metric Value'); u=h.index('Metric Unit'); k=h.index('Kernel Name')
v=[float(r[i].replace(',',''))*(1e-3 if r[u] in ('nsecond','ns') else 1) for r in rows[1:]]
print('$1 per layer', ['%.0f' % (sum(v[l::L])/len(v[l::L])) for l in range(L)], 'sum %.0f' % (sum(v)/2), [rows[1+l][k][7:20] for l in range(L)])
 "
 done
done
