"""Per-source-line stall samples of one kernel in an ncu report (needs -lineinfo + --import-source).
usage: python tools/ncu_src.py <report.ncu-rep> <kernel regex> [topN]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
# the sass,cuda view interleaves "File/Line" headers; fall back to parsing the sass view with the
# correlation column if present
rows = list(csv.reader(io.StringIO(out)))
hdr = None
tot = collections.Counter()
cur = None
samples = 0
for r in rows:
    if len(r) > 2 and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if "# Samples" not in hdr:
        continue
    try:
        s = int(r[hdr.index("# Samples")] or 0)
    except ValueError:
        continue
    src = r[hdr.index("Source")]
    tot[src.strip()[:100]] += s
    samples += s
for k, v in tot.most_common(top):
    print(f"{100 * v / max(samples, 1):5.1f}%  {k}")
