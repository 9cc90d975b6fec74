"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/launch_list.py gpurun_out/launches_c2.csv "header line" > profiles/rX_launches_c2.txt
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(lsort_dev::LevelParams.*|\(.*", "", name)
    name = name.replace("void ", "").replace("lsort_dev::", "").replace("(bool)", "").replace("(unsigned int)", "")
    return name.strip()


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = None
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000.0)
        k = short(d["Kernel Name"])
        tot[k] += us
        cnt[k] += 1
    total = sum(tot.values())
    if len(sys.argv) > 2:
        print("# " + sys.argv[2])
    print(f"# {sum(cnt.values())} launches captured (ncu serialises launches, cold caches: use shares, not absolute times)")
    print(f"# total {total / 1000:.3f} ms")
    print("# kernel  launches  total_us  share")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:62]:62s} {cnt[k]:5d} {v:10.1f} {100 * v / total:5.1f}%")


if __name__ == "__main__":
    main()
