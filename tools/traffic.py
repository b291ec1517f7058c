"""Pair the DRAM traffic of an ncu launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum; tools/prof_step.py under
--profile-from-start off) with the algorithmic bytes of the same launch
shapes (prof_step.py --profile --dump) -> profiles/traffic_<cfg>.json, the
`roofline.traffic` bench.py reports.

    python tools/traffic.py launches.csv alg.json > profiles/traffic_c3.json
"""
import collections
import csv
import json
import sys

CLASSES = (("attention", ("k_attn_tma", "k_attn_combine")), ("gemm", ("k_gemm_sk", "k_gemm_simt")),
           ("shuffle", ("k_shuffle",)))


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    alg = json.load(open(sys.argv[2]))
    hdr = None
    per = collections.defaultdict(dict)        # launch id -> metric -> value
    names = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
                 "usecond": 1, "us": 1, "msecond": 1e3}.get(unit, 1)
        per[d["ID"]][d["Metric Name"]] = v * scale
        names[d["ID"]] = d["Kernel Name"]
    out = {"_source": f"ncu launch list {sys.argv[1]} (dram__bytes_read.sum + dram__bytes_write.sum per "
                      f"launch, cold-cache, serialised) paired with {sys.argv[2]} (algorithmic bytes per "
                      f"launch of the same steady-state shape: C3 decode at {alg.get('rows')} rows)",
           "rows": alg.get("rows")}
    for cls, pats in CLASSES:
        ids = [i for i, n in names.items() if any(p in n for p in pats)]
        if cls == "attention":
            # one attention launch group = k_attn_tma (+ k_attn_combine when split)
            ids_main = [i for i in ids if "k_attn_tma" in names[i]]
            n_launch = len(ids_main)
        else:
            n_launch = len(ids)
        if not n_launch:
            continue
        dram = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in ids)
        t = sum(per[i].get("gpu__time_duration.sum", 0) for i in ids)
        a = alg.get(cls, {}).get("algorithmic_bytes_per_launch")
        out[cls] = {"dram_bytes_per_launch": dram / n_launch, "launches": n_launch,
                    "us_per_launch_ncu": t / n_launch, "algorithmic_bytes_per_launch": a,
                    "dram_over_algorithmic": (dram / n_launch / a) if a else None}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
