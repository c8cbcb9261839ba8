"""Per-level device time of one enumeration from a CC_TRACE log (library per-launch trace with
cc_options.profile = 1): paths in, records out, ms and Mpaths/ms per level and kernel kind.

    CC_TRACE=t.csv python tools/run_once.py p10x10 --profile; python tools/level_times.py t.csv
"""
import collections
import csv
import sys

rows = list(csv.DictReader(open(sys.argv[1])))
lv = collections.defaultdict(lambda: [0, 0, 0.0, 0])
tot = 0.0
for r in rows:
    if r["kind"] != "expand":
        continue
    key = int(r["level"])
    v = lv[key]
    v[0] += int(r["paths_in"])
    v[1] += int(r["children_out"])
    v[2] += float(r["ms"])
    v[3] += 1
    tot += float(r["ms"])
print(f"total expand ms {tot:.1f}, launches {sum(v[3] for v in lv.values())}")
for k in sorted(lv):
    a, b, c, nl = lv[k]
    if c > 5:
        print(f"level {k:3d} in {a:14d} out {b:14d} ms {c:8.1f} launches {nl:4d} {a / c / 1e6:6.1f} Min/ms")
