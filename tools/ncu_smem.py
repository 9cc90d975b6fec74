"""Shared-memory wavefronts (actual vs ideal) per CUDA source line of one
kernel launch in an ncu --set full report (needs -lineinfo, --import-source).

    python tools/ncu_smem.py REPORT KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kr = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kr}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, cur = "?", None, None
    agg = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            iw = hdr.index("L1 Wavefronts Shared")
            ii = hdr.index("L1 Wavefronts Shared Ideal")
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip()[:80])
            continue
        try:
            w, i = int(r[iw]), int(r[ii])
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(cur, [0, 0])
        a[0] += w
        a[1] += i
    tw = sum(a[0] for a in agg.values())
    print(f"total shared wavefronts {tw}")
    for k, (w, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        if w:
            print(f"{100 * w / max(tw, 1):5.1f}% wf {w:11d} ideal {i:11d}  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
