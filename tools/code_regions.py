"""Code bytes of one kernel between its clock64 probe marks (tools only):
python tools/code_regions.py cubin_disasm.txt kernel_substring source_file"""
import collections
import re
import sys

txt = open(sys.argv[1]).read().split('\n')
start = [i for i, l in enumerate(txt) if l.startswith('//----') and sys.argv[2] in l][0]
ins, loc = [], None
for l in txt[start + 1:]:
    if l.startswith('//----'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        loc = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s*(.*)', l)
    if m:
        ins.append((int(m.group(1), 16), loc, m.group(2)))
print('function bytes', ins[-1][0] + 16)
src = open(sys.argv[3]).read().split('\n') if len(sys.argv) > 3 else None
prev = 0
for a, loc, t in ins:
    if 'CLOCK' in t:
        line = src[loc[1] - 1].strip() if src and loc and loc[0] in sys.argv[3] else ''
        print(f"{a:#8x} (+{a - prev:6d})  {line[:70]}")
        prev = a
