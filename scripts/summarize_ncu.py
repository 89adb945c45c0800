"""Markdown summary of ncu evidence: per-kernel launch list (time share, DRAM bytes per launch)
from a --csv --metrics log, and key metrics of --set full captures. Usage:
  python scripts/summarize_ncu.py launches.csv full_a.ncu-rep [full_b.ncu-rep ...] > summary.md"""
import collections
import csv
import json
import os
import io
import re
import subprocess
import sys

UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
            per[d["ID"]][d["Metric Name"]] = v
            per[d["ID"]]["name"] = re.sub(r"\(.*", "", d["Kernel Name"]).replace("bfpp::<unnamed>::", "") \
                .replace("void ", "").strip()
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for m in per.values():
        a = agg[m["name"]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot = sum(v[1] for v in agg.values())
    g = [v for n, v in agg.items() if n.startswith("gemm")]
    if g and os.environ.get("GEMM_TRAFFIC_OUT"):  # per-launch GEMM DRAM bytes for bench.py's roofline.traffic
        c, b = sum(v[0] for v in g), sum(v[2] for v in g)
        with open(os.environ["GEMM_TRAFFIC_OUT"], "w") as f:
            json.dump({"bytes_per_launch": int(b / c), "launches_in_list": c,
                       "source": f"{path}: mean dram__bytes_read.sum + dram__bytes_write.sum over the GEMM kernel "
                                 "launches of bench.py (GPT-1.3B, N=1; weight-gradient pairs are one grouped launch)"},
                      f, indent=1)
    print("| kernel | launches | total ms | avg us | share | DRAM MB / launch |")
    print("|---|---|---|---|---|---|")
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{n}` | {c} | {t * 1e3:.2f} | {t / c * 1e6:.1f} | {t / tot:.3f} | {b / c / 1e6:.2f} |")


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[-1]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else path
    print(f"\n**`{re.sub(r'[(].*', '', name)}`** ({path.split('/')[-1]})\n")
    print("| metric | value |")
    print("|---|---|")
    for k in KEYS:
        for a, b, c in zip(h, u, v):
            if a.endswith(k) and not a.startswith(("FBSP", "TPC", "SM_C")):
                print(f"| {k} | {c} {b} |")
                break


if __name__ == "__main__":
    print("### Launch list (ncu, serialised, cold caches)\n")
    launch_list(sys.argv[1])
    print("\n### Full captures\n")
    for p in sys.argv[2:]:
        full(p)
