"""Key metrics of `ncu --set full` captures -> profiles/.

    python scripts/ncu_full_summary.py <tag> <workload> <capture.ncu-rep> [...]

Writes profiles/<tag>_ncu_full.csv (per captured launch: duration, DRAM
bytes read/written, DRAM throughput, warps active, registers, grid size)
and records the per-launch DRAM traffic of the workload's finest-level
SpMV / Vanka apply in profiles/ncu_traffic.json (keyed workload -> kernel,
read by bench.py as roofline.traffic).  Convention: the capture's last
launch of each kernel kind is the finest-level one (captures are taken with
-k / -s / -c selecting finest-level launches).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "lts__t_sectors_srcunit_tex_op_read.sum"]
TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{k: (r[hdr.index(k)], units[hdr.index(k)]) for k in KEYS if k in hdr} for r in rows[2:]]


def kind(name):
    if "spmv" in name:
        return "spmv"
    if "vanka_apply" in name:
        return "vanka_apply"
    return None


def main():
    tag, workload, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    recs = []
    for rep in reps:
        recs += rows_of(rep)
    path = os.path.join(PROF, f"{tag}_ncu_full.csv")
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + KEYS[1:] + ["dram_bytes_per_launch"])
        traffic = {}
        for r in recs:
            name = r["Kernel Name"][0].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            rd = float(r["dram__bytes_read.sum"][0]) * TO_BYTES[r["dram__bytes_read.sum"][1]]
            wr = float(r["dram__bytes_write.sum"][0]) * TO_BYTES[r["dram__bytes_write.sum"][1]]
            w.writerow([name] + [r[k][0] + " " + r[k][1] for k in KEYS[1:] if k in r] + [rd + wr])
            if kind(name):
                traffic[kind(name)] = rd + wr
    tpath = os.path.join(PROF, "ncu_traffic.json")
    data = json.load(open(tpath)) if os.path.exists(tpath) else {}
    if "spmv" in data and not isinstance(data["spmv"], dict):     # round-1 flat layout
        data = {"3d_large": {k: v for k, v in data.items() if k != "source"},
                "source": {"3d_large": data.get("source")}}
    data.setdefault(workload, {}).update(traffic)
    data.setdefault("source", {})[workload] = f"profiles/{tag}_ncu_full.csv"
    json.dump(data, open(tpath, "w"), indent=1)
    print(open(path).read())


if __name__ == "__main__":
    main()
