"""Quick look at an ncu report: key metrics, stall reasons, hottest SASS."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__grid_size', 'launch__registers_per_thread', 'lts__t_bytes.sum']
for r in rows[2:]:
    print(' | '.join(f"{w.split('__')[1][:38]}={r[h.index(w)]}" for w in want if w in h))
r = rows[2]
st = [(float(r[i].replace(',', '')), k) for i, k in enumerate(h) if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued') and r[i].replace(',', '').replace('.', '').isdigit()]
print(sorted(st, reverse=True)[:8])
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    blocks = []; cur = None
    for r in rows:
        if r and r[0] == 'Kernel Name':
            cur = [r[1], None, []]; blocks.append(cur); continue
        if r and r[0] == 'Address': cur[1] = r; continue
        if cur and cur[1] and len(r) > 5: cur[2].append(r)
    name, hh, data = blocks[0]
    iS = hh.index('Warp Stall Sampling (All Samples)'); iE = hh.index('Instructions Executed')
    tot = sum(int(x[iS]) for x in data)
    print('samples', tot)
    for x in sorted(data, key=lambda x: -int(x[iS]))[:int(sys.argv[2])]:
        print(x[0][-5:], x[iS].rjust(5), x[iE].rjust(8), x[1].strip()[:90])
    op = collections.Counter()
    for x in data:
        o = x[1].strip().split()
        if not o: continue
        o = o[1] if o[0].startswith('@') else o[0]
        op[o.split('.')[0]] += int(x[iE])
    print(op.most_common(16))
