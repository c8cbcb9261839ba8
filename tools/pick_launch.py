"""Index (among expand launches) of the largest launch in a CC_TRACE log (for ncu -s)."""
import csv
import sys

rows = [r for r in csv.DictReader(open(sys.argv[1])) if r["kind"] == "expand"]
print(max(range(len(rows)), key=lambda i: int(rows[i]["paths_in"])))
