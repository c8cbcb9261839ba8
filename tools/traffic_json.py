"""Write profiles/ncu_traffic.json: DRAM traffic of one ncu --set full capture of the dominant
kernel next to the algorithmic bytes of the same launch (from the CC_TRACE log of the same run).
bench.py reports the pair as roofline.traffic / traffic_over_alg.

    python tools/traffic_json.py p10x10 gpurun_out/prof44.ncu-rep gpurun_out/trace44.csv \
        --level 44 --kernel 'k_expand_fq<2>' --record-bytes 24 --r-alg 16

The captured launch is the first expansion of --level (ncu --nvtx-include "expand L<t> f<fuse>/"
-c 1, tools/r02_prof44.sh).  Records: a two-level launch reads F_t and writes F_{t+2}; a
level-synchronous expansion of the same paths would also write and read F_{t+1}
(records_levelsync = in + 2 * next + out).
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
ap.add_argument("--level", type=int, nargs="+", required=True, help="level(s) of the captured launch")
ap.add_argument("--kernel", required=True)
ap.add_argument("--record-bytes", type=int, required=True)
ap.add_argument("--r-alg", type=int, required=True, help="SURVEY 8(d) R_alg of the workload")
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_traffic.json"))
a = ap.parse_args()

raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))


def metric(k):
    return float(d[k]) * SCALE[u[k]]


dram = metric("dram__bytes_read.sum") + metric("dram__bytes_write.sum")
dur_ms = metric("gpu__time_duration.sum")
expands = [r for r in csv.DictReader(open(a.trace)) if r["kind"] == "expand" and int(r["level"]) in a.level]
row = expands[0]
slots_in, slots_out = int(row["paths_in"]), int(row["children_out"])
pin, pnext, pout = int(row["paths_real"]), int(row["paths_next"]), int(row["out_real"])
two = int(row["fuse"]) == 2
levelsync = pin + pout + (2 * pnext if two else 0)
path = a.out
data = json.load(open(path)) if os.path.exists(path) else {}
data[a.workload] = {
    "kernel": a.kernel, "launch": f"first expansion of level {row['level']} (fuse {row['fuse']})",
    "paths_in": pin, "paths_next": pnext if two else 0, "records_out": pout,
    "slots_in": slots_in, "slots_out": slots_out, "record_bytes": a.record_bytes,
    "records_levelsync": levelsync, "r_alg": a.r_alg,
    "bytes_moved": (slots_in + slots_out) * a.record_bytes, "bytes_alg": levelsync * a.r_alg,
    "dram_bytes": dram, "dram_over_moved": dram / ((slots_in + slots_out) * a.record_bytes),
    "dram_over_alg": dram / (levelsync * a.r_alg), "duration_ms": dur_ms,
    "source": f"{os.path.basename(a.report)} + {os.path.basename(a.trace)}",
}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[a.workload]))
