"""Bucket ncu SASS samples/executions of the first kernel in a report into
contiguous regions (split at large jumps of the execution count)."""
import csv, subprocess, sys
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
blocks = []; cur = None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = [r[1], None, []]; blocks.append(cur); continue
    if r and r[0] == 'Address': cur[1] = r; continue
    if cur and cur[1] and len(r) > 5: cur[2].append(r)
name, h, data = blocks[int(sys.argv[2]) if len(sys.argv) > 2 else 0]
iS = h.index('Warp Stall Sampling (All Samples)'); iE = h.index('Instructions Executed')
tot_s = sum(int(x[iS]) for x in data); tot_e = sum(int(x[iE]) for x in data)
# regions: marked by labels we recognise
reg = []
for x in data:
    a = x[0][-5:]; op = x[1].strip()
    reg.append((a, int(x[iS]), int(x[iE]), op))
# print a compact listing: every instruction with >= 0.5% of samples, plus running totals
acc_s = 0
for a, s, e, op in reg:
    acc_s += s
    if s >= 0.006 * tot_s or 'SYNCS' in op or 'BAR' in op or 'EXIT' in op or 'REDG' in op:
        print(f"{a} {s:5d} {e:8d} cum={100*acc_s/tot_s:5.1f}%  {op[:70]}")
print('samples', tot_s, 'instrs', tot_e)
