"""Summarise an ncu --csv launch list: per-kernel count / mean / share."""
import csv, io, sys, collections
txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
agg = collections.OrderedDict()
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "")[:48]
    v = float(r["Metric Value"])
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += v
tot = sum(a[1] for a in agg.values())
for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} n={n:4d} mean={s/n/1e3:9.2f}us share={100*s/tot:5.1f}%")
