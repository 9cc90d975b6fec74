"""Per-CUDA-source-line instruction counts and stall samples of one kernel
launch in an ncu report (needs -lineinfo and --import-source on).

    python tools/ncu_lines.py REPORT KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kr = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kr}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr = "?", None
    agg = {}
    cur = None
    tot_i = tot_s = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            iw = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0]:  # source line row
            cur = (fname, int(r[0]), r[1].strip()[:90])
            continue
        try:
            i, w = int(r[ie]), int(r[iw])
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(cur, [0, 0])
        a[0] += i
        a[1] += w
        tot_i += i
        tot_s += w
    print(f"total warp-inst {tot_i}  samples {tot_s}")
    for k, (i, w) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*i/max(tot_i,1):5.1f}% inst {100*w/max(tot_s,1):5.1f}% samp  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
