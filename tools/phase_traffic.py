"""DRAM traffic per sort phase from an ncu metrics CSV of tools/profile_sort.py.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file T.csv python tools/profile_sort.py DIST N 1
    python tools/phase_traffic.py T.csv N > profiles/rX_kernel_traffic.json
"""
import collections
import csv
import json
import sys

PHASE = [("k_base", "base"), ("k_small_sort", "base"), ("k_scatter", "scatter"), ("k_direct<", "scatter"), ("k_hist", "classify"),
         ("k_fill", "fill"), ("k_verify", None)]


def phase_of(name):
    for pre, ph in PHASE:
        if name.startswith(pre):
            return ph
    return "models"


def main():
    path, n = sys.argv[1], int(float(sys.argv[2]))
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("lsort_dev::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        per[(d["ID"], name)][d["Metric Name"]] = v * scale
    agg = collections.defaultdict(lambda: {"dram_bytes": 0.0, "ns": 0.0, "launches": 0})
    for (_, name), m in per.items():
        ph = phase_of(name)
        if ph is None:
            continue
        a = agg[ph]
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a["ns"] += m.get("gpu__time_duration.sum", 0)
        a["launches"] += 1
    out = {"source": path, "keys": n, "note": "ncu per-kernel DRAM counters summed per sort phase, one sort",
           "phases": {k: {"dram_bytes": v["dram_bytes"], "dram_bytes_per_key": v["dram_bytes"] / n,
                          "launches": v["launches"], "ncu_ms": v["ns"] / 1e6} for k, v in agg.items()}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
