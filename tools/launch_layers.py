"""Per-layer average of a kernel's launches in an ncu launch-list CSV
(launches in order; layer = launch index mod depth)."""
import csv, sys
path, kernel, depth = sys.argv[1], sys.argv[2], int(sys.argv[3])
rows = list(csv.reader(open(path)))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
v = []
for r in rows[start:]:
    if kernel in r[ik]:
        x = float(r[iv].replace(",", ""))
        v.append(x / 1e3 if r[iu] in ("nsecond", "ns") else (x * 1e3 if r[iu] in ("msecond", "ms") else x))
print(kernel, "launches", len(v), "per layer (us):", ["%.1f" % (sum(v[l::depth]) / max(1, len(v[l::depth]))) for l in range(depth)])
