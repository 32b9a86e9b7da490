"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] and r[0].isdigit():
        line = (cur, int(r[0]))
        agg[line][3] = r[1].strip()[:70]
    try:
        s, n, t = int(r[4]), int(r[7]), int(r[8])
    except (ValueError, IndexError):
        continue
    a = agg[line]
    a[0] += s
    a[1] += n
    a[2] += t
ts = sum(a[0] for a in agg.values())
ti = sum(a[1] for a in agg.values())
print("samples", ts, "warp insts", ti)
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:<4} {a[3]:<70} smp {100*a[0]/ts:5.1f}% inst {100*a[1]/ti:5.1f}% thr/inst {a[2]/max(1,a[1]):.1f}")
