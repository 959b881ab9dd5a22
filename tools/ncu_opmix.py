"""Opcode mix and stall samples of one kernel from `ncu --page source --csv --print-source sass`.
usage: python tools/ncu_opmix.py <source.csv> [topN]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
op, st = collections.Counter(), collections.Counter()
h = None
for r in rows:
    if "Source" in r and "Instructions Executed" in r:
        h = r
        iS, iE, iSm = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or len(r) < len(h):
        continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
    if not m or not r[iE].isdigit():
        continue
    op[m.group(2)] += int(r[iE])
    st[m.group(2)] += int(r[iSm] or 0)
tot, totS = sum(op.values()), max(sum(st.values()), 1)
print("total warp instructions", tot)
for o, n in op.most_common(top):
    print(f"{o:10s} {n / tot * 100:5.1f}%   stall samples {st[o] / totS * 100:5.1f}%")
