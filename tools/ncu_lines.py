"""Summarise an ncu `--page source --print-source cuda,sass --csv` dump by CUDA line:
stall samples and executed instructions per source line (file:line)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file = "?"
by_line = collections.Counter()
inst_line = collections.Counter()
src = {}
tot = 0.0
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    try:
        v = float(r[4] or 0)
        ins = float(r[7] or 0)
    except ValueError:
        continue
    if r[0]:
        key = f"{cur_file}:{r[0]}"
        src[key] = r[1].strip()[:80]
        cur = key
    else:
        continue
    by_line[cur] += v
    inst_line[cur] += ins
    tot += v
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k, v in by_line.most_common(n):
    print(f"{100 * v / max(tot, 1):5.1f}%  inst={inst_line[k]:.3g}  {k:18s} {src.get(k, '')}")
