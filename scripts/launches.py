"""Summarise an ncu --csv launch list: mean duration per kernel name."""
import csv, io, sys, collections
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); gi = h.index('Grid Size')
acc = collections.OrderedDict()
for r in rows[1:]:
    key = (r[ki].split('(')[0][:40], r[gi])
    acc.setdefault(key, []).append(float(r[vi]) / 1000.0)
for (k, g), v in acc.items():
    print(f"{k:42s} {g:>16s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us  min={min(v):8.2f}")
