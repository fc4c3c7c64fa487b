"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time per kernel name."""
import csv, collections, sys
rows = list(csv.DictReader([l for l in open(sys.argv[1]) if l.startswith('"')]))
d = collections.OrderedDict()
for r in rows:
    k = r['Kernel Name'].split('(')[0]
    d.setdefault(k, []).append(float(r['Metric Value']) / 1e3)
tot = sum(sum(v) for v in d.values())
for k, v in d.items():
    print(f"{k:50s} n={len(v):4d} sum={sum(v):10.1f}us mean={sum(v)/len(v):9.1f}us share={sum(v)/tot:.3f}")
