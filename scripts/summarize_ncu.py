"""Summarise ncu outputs into profiles/ (tracked).

    python scripts/summarize_ncu.py launches gpurun_out/launches.csv profiles/r01_launches_c3_step4.md
    python scripts/summarize_ncu.py full gpurun_out/attn.ncu-rep profiles/r01_attn_spatial_ncu.json
"""

import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
]


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")[:80]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{name}` | {n} | {us:.0f} | {100 * us / tot:.1f}% |")
    out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.0f} | 100% |")
    text = "\n".join(out) + "\n"
    open(dst, "w").write(text)
    print(text)


def full(src, dst):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    # ncu scales units per value (Mbyte / Gbyte, us / ms): normalise bytes to MB, time to us
    to_base = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
               "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:90]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    d[m] = float(r[i].replace(",", "")) * to_base.get(units[i], 1.0)
                except ValueError:
                    d[m] = r[i]
        d["units"] = "bytes in MB, durations in us"
        res.append(d)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
