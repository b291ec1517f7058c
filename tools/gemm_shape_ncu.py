"""Summarise tools/gemm_shape_ncu.sh captures: one CSV row per (GEMM, rows).

    python tools/gemm_shape_ncu.py gpurun_out/x > profiles/<round>_gemm_per_shape_ncu.csv
"""
import csv
import glob
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6535.0
NAMES = {"in": "merged QKV+FFN-up (N=28672,K=4096)", "out": "merged attn-out+FFN-down (N=4096,K=20480)",
         "lm": "LM head + argmax (N=50400,K=4096)"}
WBYTES = {"in": 28672 * 4096 * 2, "out": 4096 * 20480 * 2, "lm": 50400 * 4096 * 2}
print("gemm,rows,launches,us_mean,dram_MB_per_launch,weight_MB,dram_GBps,frac_of_measured_copy_peak_%.0f,"
      "ncu_dram_pct_of_peak,tensor_pipe_active_pct" % peak)
rows = []
for f in glob.glob(os.path.join(sys.argv[1], "gemm_shape_*_*.csv")):
    part, M = re.match(r".*gemm_shape_(\w+?)_(\d+)\.csv", f).groups()
    met = defaultdict(dict)
    with open(f) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        name = r["Metric Name"]
        if name.startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        if name == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(unit, 1)
        met[r["ID"]][name] = v
    if not met:
        continue
    n = len(met)
    us = sum(m["gpu__time_duration.sum"] for m in met.values()) / n
    by = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in met.values()) / n
    dp = sum(m["dram__throughput.avg.pct_of_peak_sustained_elapsed"] for m in met.values()) / n
    tp = sum(m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"] for m in met.values()) / n
    gbs = by / (us * 1e-6) / 1e9
    rows.append((list(NAMES).index(part), int(M), f'"{NAMES[part]}",{M},{n},{us:.1f},{by / 1e6:.1f},'
                 f'{WBYTES[part] / 1e6:.1f},{gbs:.0f},{gbs / peak:.3f},{dp:.1f},{tp:.1f}'))
for _, _, line in sorted(rows):
    print(line)
