"""Summarise an `ncu --page source --csv --print-source sass` export:
per kernel (first occurrence), total stall samples, stall-reason split and
the hottest SASS instructions.  usage: python tools/ncu_source_summary.py file.csv [top]"""
import csv
import re
import sys
from collections import Counter


def main(path, top=25, only=None):
    kern, hdr, seen = None, None, set()
    stats = {}
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "Kernel Name":
            kern = row[1]
            hdr = None
            continue
        if row[0] == "Address":
            hdr = row
            continue
        if hdr is None or kern is None:
            continue
        key = re.sub(r"\(.*", "", kern)
        if only and only not in key:
            continue
        st = stats.setdefault(kern, {"n": 0, "stall": Counter(), "ins": [], "id": len(stats)})
        d = dict(zip(hdr, row))
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        st["n"] += s
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                v = d.get(h, "0")
                if v and v != "0":
                    st["stall"][h] += int(v)
        st["ins"].append((s, d["Address"][-5:], d["Source"].strip()[:90]))
    done = set()
    for kern, st in stats.items():
        short = re.sub(r"\(.*", "", kern)
        if short in done:
            continue
        done.add(short)
        print(f"=== {short}  samples={st['n']}")
        tot = max(st["n"], 1)
        print("   stalls:", ", ".join(f"{k[6:]} {100*v/tot:.0f}%" for k, v in st["stall"].most_common(8)))
        for s, a, src in sorted(st["ins"], key=lambda x: -x[0])[:top]:
            print(f"   {s:6d} {100*s/tot:5.1f}% {a} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, sys.argv[3] if len(sys.argv) > 3 else None)
