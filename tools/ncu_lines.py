"""Aggregate an ncu source page (--print-source=cuda,sass --csv) per CUDA source line:
warp instructions executed and stall samples, to see where a kernel's instructions go.

    ncu -i rep --page source --csv --print-source=cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
inst = collections.Counter()
samp = collections.Counter()
text = {}
cur = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r) if k not in ("Source",)}
        ii = r.index("Instructions Executed")
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = int(r[0])
        text[cur] = r[1][:90]
        continue
    try:
        inst[cur] += int(r[ii])
        samp[cur] += int(r[si])
    except ValueError:
        pass
ti = sum(inst.values())
ts = sum(samp.values())
print(f"total warp instructions {ti}, stall samples {ts}")
for ln, v in inst.most_common(top):
    print(f"{ln:5d} {v / ti:6.1%} inst {samp[ln] / ts:6.1%} samples  {text.get(ln, '')}")
