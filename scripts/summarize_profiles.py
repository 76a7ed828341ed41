"""Turn one round's ncu captures (gpurun_out/) into the tracked summaries under profiles/
(development tool, runs on the CPU box): launch-list shares, the per-kernel `--set full`
summary and the per-launch DRAM traffic that bench.py reports as roofline.traffic.

    python scripts/summarize_profiles.py r1c   # reads gpurun_out/launches_r1c.csv, prof_r1c.ncu-rep
"""

import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
ALG = {"k_fused_ldg<1, 0": ("fused", 32.5), "k_fused_ldg<1, 2": ("fused_local", 28.25),
       "k_apply_quant<1>": ("apply_quant", 16.25)}
N50 = 25557032


def short(name: str) -> str:
    m = re.search(r"(k_\w+<[^>]*>|k_\w+)", name)
    return m.group(1) if m else name[:60]


def launches(tag):
    rows = [l for l in open(os.path.join(OUT, f"launches_{tag}.csv")) if l.startswith('"')]
    r = csv.reader(io.StringIO("".join(rows)))
    h = next(r)
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = defaultdict(lambda: [0, 0.0])
    allk = []
    for row in r:
        ns = float(row[vi])
        k = short(row[ki]) if "cdsgd" in row[ki] or row[ki].startswith("void k_") or "k_" in row[ki][:40] else "torch/other"
        per[k][0] += 1
        per[k][1] += ns / 1e3
        allk.append((k, ns / 1e3))
    ours = {k: v for k, v in per.items() if k.startswith("k_")}
    tot = sum(v[1] for v in ours.values())
    return {k: {"launches": v[0], "total_us": round(v[1], 1), "avg_us": round(v[1] / v[0], 1),
                "share_of_our_kernels": round(v[1] / tot, 3)} for k, v in sorted(ours.items(), key=lambda x: -x[1][1])}


def full(tag):
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(txt))
    h = next(r)
    units = next(r)
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    want = {"gpu__time_duration.sum": "gpu_time_us", "dram__bytes_read.sum": "dram_read_MB",
            "dram__bytes_write.sum": "dram_write_MB", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
            "launch__registers_per_thread": "regs", "launch__grid_size": "grid", "launch__block_size": "block",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
            "smsp__inst_executed.sum": "inst_executed", "sm__cycles_active.avg": "sm_cycles_active_avg",
            "sm__cycles_active.max": "sm_cycles_active_max", "gpc__cycles_elapsed.max": "cycles_elapsed"}
    out = []
    for row in r:
        d = {"kernel": row[h.index("Kernel Name")][:40]}
        for m, k in want.items():
            if m in h and row[h.index(m)]:
                i = h.index(m)
                d[k] = float(row[i].replace(",", "")) * scale.get(units[i], 1.0)  # MB / us where dimensioned
        out.append(d)
    return out


def main():
    tag = sys.argv[1]
    L = launches(tag)
    F = full(tag)
    json.dump({"source": f"gpurun_out/launches_{tag}.csv (ncu --metrics gpu__time_duration.sum --clock-control none; "
                         "cold-cache, serialised)", "kernels": L},
              open(os.path.join(PROF, f"{tag}_ncu_launch_shares.json"), "w"), indent=1)
    json.dump(F, open(os.path.join(PROF, f"{tag}_ncu_full_summary.json"), "w"), indent=1)
    traffic = {"_note": f"dram__bytes_read.sum + dram__bytes_write.sum per launch from `ncu --set full --clock-control none` "
                        f"(cold L2, serialised replay) of the bench command, capture {tag}. Writes can fall below the "
                        "algorithmic bytes: part of a kernel's output is still dirty in the 126 MB L2 when it ends.",
               "resnet50": {}}
    tp = os.path.join(PROF, "ncu_traffic.json")
    if os.path.exists(tp):  # keep classes this capture did not include
        traffic["resnet50"].update(json.load(open(tp)).get("resnet50", {}))
    for d in F:
        for pat, (cls, bpe) in ALG.items():
            if d["kernel"].startswith("void " + pat) and traffic["resnet50"].get(cls, {}).get("_capture") != tag:
                traffic["resnet50"][cls] = {"kernel": d["kernel"],
                                            "dram_bytes_per_launch": int(1e6 * (d["dram_read_MB"] + d["dram_write_MB"])),
                                            "algorithmic_bytes": int(bpe * N50),
                                            "gpu_time_us_cold": d["gpu_time_us"], "_capture": tag}
    json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    print(json.dumps(L, indent=1))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
