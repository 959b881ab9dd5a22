"""Stall-reason breakdown of selected source lines of one kernel (ncu --page source sass CSV + the
nvdisasm -g listing of the same binary).  usage: python tools/ncu_line_stalls.py src.csv fn.sass file:line ..."""
import collections
import csv
import re
import sys

csvf, sassf = sys.argv[1], sys.argv[2]
want = [(a.split(':')[0], int(a.split(':')[1])) for a in sys.argv[3:]]
cur, amap = None, {}
for ln in open(sassf):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
h = rows[1]
stalls = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
agg = collections.defaultdict(collections.Counter)
base = None
for r in rows[2:]:
    try:
        a = int(r[0], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    key = amap.get(a - base, ('?', 0))
    for c in stalls:
        agg[key][c] += int(r[h.index(c)] or 0)
for k in want:
    s = sum(agg[k].values())
    print(k, s, {a: round(100 * v / max(s, 1)) for a, v in agg[k].most_common(4)})
