"""Summarise ncu outputs into small text files for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  > profiles/r01_x.txt
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {rep}")
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"\n## kernel: {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in d:
                print(f"{k:60s} {d[k]:>20s} {u.get(k, '')}")
        try:
            rd = float(d["dram__bytes_read.sum"]) * (1e9 if u["dram__bytes_read.sum"] == "Gbyte" else 1e6 if u["dram__bytes_read.sum"] == "Mbyte" else 1)
            wr = float(d["dram__bytes_write.sum"]) * (1e9 if u["dram__bytes_write.sum"] == "Gbyte" else 1e6 if u["dram__bytes_write.sum"] == "Mbyte" else 1)
            t = float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "ms" else 1e-6 if u["gpu__time_duration.sum"] == "us" else 1e-9)
            print(f"{'dram traffic (read+write) bytes':60s} {rd + wr:20.4e}")
            print(f"{'dram traffic / duration (GB/s)':60s} {(rd + wr) / t / 1e9:20.1f}")
        except (KeyError, ValueError, ZeroDivisionError):
            pass
    # stall breakdown from the source page
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    stalls = collections.Counter()
    hdr = None
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "Line No":
            hdr = {k: i for i, k in enumerate(r)}
            continue
        if hdr and len(r) > 7 and r[2]:
            for k, i in hdr.items():
                if k.startswith("stall_") and "Not Issued" not in k:
                    try:
                        stalls[k] += int(r[i])
                    except (ValueError, IndexError):
                        pass
    tot = sum(stalls.values())
    if tot:
        print("\n## warp stall samples (share)")
        for k, v in stalls.most_common(10):
            print(f"{k:40s} {v / tot:7.1%}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = {k: i for i, k in enumerate(r)}
            continue
        if not hdr or len(r) < len(hdr):
            continue
        if r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[hdr["Kernel Name"]].split("(")[0]
        val = float(r[hdr["Metric Value"]].replace(",", ""))
        unit = r[hdr["Metric Unit"]]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        per[name][0] += 1
        per[name][1] += val * scale
    tot = sum(v[1] for v in per.values())
    print(f"# ncu launch list {path}: {sum(v[0] for v in per.values())} launches, {tot:.3f} ms total (serialised, cold-cache)")
    print(f"{'kernel':60s} {'launches':>9s} {'ms':>12s} {'share':>7s}")
    for k, (n, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:9d} {ms:12.3f} {ms / tot:7.1%}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
