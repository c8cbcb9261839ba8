"""Write profiles/ncu_traffic.json: DRAM traffic of one ncu --set full capture of the dominant
kernel next to the algorithmic bytes of the same launch (from a CC_TRACE log of the same
deterministic run).  bench.py reports the pair as roofline.traffic / traffic_over_alg.

    python tools/traffic_json.py p10x10 gpurun_out/prof.ncu-rep gpurun_out/trace.csv \
        --launch 45 --kernel 'k_expand_blocked<2,3,1,0>' --record-bytes 24
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("report")
ap.add_argument("trace")
ap.add_argument("--launch", type=int, required=True, help="0-based index among the expand launches")
ap.add_argument("--kernel", required=True)
ap.add_argument("--record-bytes", type=int, required=True)
a = ap.parse_args()

raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))


def metric(k):
    return float(d[k]) * SCALE[u[k]]


dram = metric("dram__bytes_read.sum") + metric("dram__bytes_write.sum")
dur_ms = metric("gpu__time_duration.sum")
expands = [r for r in csv.DictReader(open(a.trace)) if r["kind"] == "expand"]
row = expands[a.launch]
paths_in, out = int(row["paths_in"]), int(row["children_out"])
alg = (paths_in + out) * a.record_bytes
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[a.workload] = {
    "kernel": a.kernel, "launch": f"expand launch #{a.launch + 1} (ncu -k regex:... -s {a.launch} -c 1)",
    "paths_in": paths_in, "children_out": out, "record_bytes": a.record_bytes, "alg_bytes": alg,
    "dram_bytes": dram, "dram_over_alg": dram / alg, "duration_ms": dur_ms,
    "source": f"{os.path.basename(a.report)} + {os.path.basename(a.trace)}",
}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[a.workload]))
