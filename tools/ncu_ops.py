"""Instruction-mix and stall hot spots of one kernel launch in an ncu report.

    python tools/ncu_ops.py REPORT KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep, kr = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kr}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[0][:2])
    hdr = rows[1]
    ia, ie, iw = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for i, r in enumerate(rows[2:]):
        try:
            data.append((int(r[ie]), int(r[iw]), i, r[ia].strip()))
        except (ValueError, IndexError):
            pass
    half = len(data) // 2
    if half and [d[3] for d in data[:half]] == [d[3] for d in data[half:2 * half]]:
        data = data[:half]
    tot = sum(d[0] for d in data) or 1
    totw = sum(d[1] for d in data) or 1
    print("total warp-inst", tot, "samples", totw)
    c, cs = Counter(), Counter()
    for e, w, i, src in data:
        tok = src.split()
        op = tok[1] if tok and tok[0].startswith("@") and len(tok) > 1 else (tok[0] if tok else "?")
        op = op.split(".")[0]
        c[op] += e
        cs[op] += w
    for op, v in c.most_common(top):
        print(f"  {op:10s} {100*v/tot:5.1f}% inst  {100*cs[op]/totw:5.1f}% samples")
    print("hottest lines:")
    for e, w, i, src in sorted(data, key=lambda x: -x[1])[:12]:
        print(f"  {i:6d} exec={e:>10d} samp={w:>6d}  {src[:70]}")


if __name__ == "__main__":
    main()
