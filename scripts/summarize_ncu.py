"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python scripts/summarize_ncu.py <tag> <launches.csv> [<full.ncu-rep>]

Writes profiles/<tag>_launch_shares.csv (per-kernel launches, device time
and share of the profiled program, cold-cache serialised times from
`ncu --metrics gpu__time_duration.sum`), profiles/<tag>_ncu_full.csv (the
key `--set full` metrics of the captured launches) and updates
profiles/ncu_traffic.json (DRAM bytes per application of the two dominant
kernels, read by bench.py as roofline.traffic).
"""
import collections
import csv
import gzip
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def short(name):
    return name.split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("unnamed>::", "").replace(
        "alefsi::", "")


def launch_shares(tag, path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[h + 1:]:
        v = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        tot[short(r[ki])] += v
        cnt[short(r[ki])] += 1
    T = sum(tot.values())
    out = os.path.join(PROF, f"{tag}_launch_shares.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_ms", "avg_ms", "share"])
        for k, v in tot.most_common():
            w.writerow([k, cnt[k], f"{v:.4f}", f"{v / cnt[k]:.5f}", f"{v / T:.4f}"])
    with open(path, "rb") as src, gzip.open(os.path.join(PROF, f"{tag}_launches.csv.gz"), "wb") as dst:
        shutil.copyfileobj(src, dst)
    print(open(out).read())


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "launch__grid_size", "launch__block_size"]


def full_metrics(tag, rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    cols = [w for w in WANT if w in hdr]
    out = os.path.join(PROF, f"{tag}_ncu_full.csv")
    traffic = {}
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + [f"{c} [{units[hdr.index(c)]}]" for c in cols])
        for r in rows[2:]:
            name = short(r[hdr.index("Kernel Name")])
            vals = [r[hdr.index(c)] for c in cols]
            w.writerow([name] + vals)
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            ur = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = rd * ur[units[hdr.index("dram__bytes_read.sum")]] + \
                wr * ur[units[hdr.index("dram__bytes_write.sum")]]
            kind = "spmv" if name.startswith("spmv") else (
                "vanka_apply" if name.startswith("vanka_apply") else name)
            traffic.setdefault(kind, []).append(b)
    print(open(out).read())
    path = os.path.join(PROF, "ncu_traffic.json")
    cur = json.load(open(path)) if os.path.exists(path) else {}
    # spmv: one launch per application; vanka: one launch per patch group
    # (fluid, solid) -> the largest plus the smallest captured launch
    if "spmv" in traffic:
        cur["spmv"] = max(traffic["spmv"])
    if "vanka_apply" in traffic:
        v = sorted(traffic["vanka_apply"])
        cur["vanka_apply"] = v[-1] + (v[0] if len(v) > 1 and v[0] < 0.5 * v[-1] else 0.0)
    cur["source"] = f"profiles/{tag}_ncu_full.csv (ncu --set full, dram__bytes_read+write)"
    json.dump(cur, open(path, "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1]
    launch_shares(tag, sys.argv[2])
    if len(sys.argv) > 3:
        full_metrics(tag, sys.argv[3])
