"""Per-SASS-instruction execution counts of an ncu source page (--print-source=sass --csv),
normalised by a reference count (e.g. the executions of the tile loop's first instruction),
to read a kernel's instruction budget per tile.

    python tools/ncu_sass.py src_sass.csv [norm]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    try:
        out.append((r[hdr["Address"]], r[hdr["Source"]].strip(), int(r[hdr["Instructions Executed"]]),
                    int(r[hdr["Warp Stall Sampling (All Samples)"]])))
    except (ValueError, KeyError):
        pass
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot = sum(x[2] for x in out)
print(f"# {len(out)} SASS instructions, {tot} executed, {tot / norm:.1f} per norm unit")
for a, s, n, st in out:
    print(f"{a[-5:]} {n / norm:8.2f} {st:6d}  {s}")
