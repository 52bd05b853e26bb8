"""Per-kernel summary of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
agg = collections.defaultdict(list)
for r in rows[1:]:
    try:
        agg[(r[ki].split("(")[0][:60], r[gi], r[bi])].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
tot = sum(sum(v) for v in agg.values())
print(f"{'n':>5} {'avg_us':>9} {'share':>6}  kernel [grid x block]")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):5d} {sum(v)/len(v)/1000:9.2f} {100*sum(v)/tot:5.1f}%  {k[0]} [{k[1]} x {k[2]}]")
