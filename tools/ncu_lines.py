"""Attribute ncu SASS-level samples/instructions to source lines (uses nvdisasm -g line info).
usage: python tools/ncu_lines.py <ncu-source-page.csv> <function.sass (nvdisasm -g)> [topN]"""
import collections
import csv
import re
import sys

csvf, sassf = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = None
amap = {}
for ln in open(sassf):
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
hdr = rows[1]
ai, ns, ie = hdr.index('Address'), hdr.index('# Samples'), hdr.index('Thread Instructions Executed')
base = None
bl, bi = collections.Counter(), collections.Counter()
tot = toti = 0
for r in rows[2:]:
    try:
        a = int(r[ai], 16)
        s = int(r[ns] or 0)
        e = int(r[ie] or 0)
    except Exception:
        continue
    if base is None:
        base = a
    key = amap.get(a - base, ('?', 0))
    bl[key] += s
    bi[key] += e
    tot += s
    toti += e
print('samples', tot, 'thread instr %.3g' % toti)
src = {}
import os
for f in os.listdir('paper_2312_07874_b200/csrc'):
    src[f] = open('paper_2312_07874_b200/csrc/' + f).read().split('\n')
for key, s in bl.most_common(top):
    f, l = key
    text = src[f][l - 1].strip()[:88] if f in src and 0 < l <= len(src[f]) else ''
    print(f'{100 * s / tot:5.1f}% smp {100 * bi[key] / toti:5.1f}% ins {f}:{l}  {text}')
