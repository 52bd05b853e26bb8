"""Stall samples of an ncu SASS source export (tools/_ncu1.sh *_source.csv)
split at barriers / mbarrier waits: where a kernel's time goes by phase.
usage: python tools/ncu_segments.py file.csv"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if r and r[0] == "Address"][0]
ins = [dict(zip(hdr, r)) for r in rows if r and r[0].startswith("0x")]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
seg, acc, exe, fp, n, start = Counter(), 0, 0, 0, 0, ins[0]["Address"]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in ins)
print("total samples", tot)
for d in ins:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    acc += s
    n += 1
    for h in stalls:
        seg[h] += int(d[h] or 0)
    e = int(d["Instructions Executed"] or 0)
    exe += e
    txt = d["Source"].strip()
    if re.search(r"\b(DADD|DMUL|DFMA)\b", txt):
        fp += e
    if "BAR.SYNC" in txt or ("SYNCS" in txt and "TRYWAIT" in txt) or txt.startswith("EXIT") or txt.startswith("RET"):
        top = ", ".join(f"{k[6:]}:{v}" for k, v in seg.most_common(5))
        print(f"{start[-5:]}..{d['Address'][-5:]} n={n:5d} samp={acc:5d} ({100*acc/max(tot,1):4.1f}%) fp64={fp:8d} | {top} | {txt[:34]}")
        acc = exe = n = fp = 0
        start = d["Address"]
        seg = Counter()
