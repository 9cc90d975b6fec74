"""Summarise an ncu report: per kernel launch the key throughput metrics.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--stalls]
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("Kernel Name", "kernel"), ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "occ_reg"), ("launch__occupancy_limit_shared_mem", "occ_smem"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("smsp__inst_executed.sum", "inst"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conf"),
    ("lts__t_sectors_op_write.sum", "l2_wr_sectors"),
]
STALLS = ["smsp__average_warp_latency_issue_stalled_", "smsp__pcsamp_warps_issue_stalled_"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        parts = []
        for m, short in WANT:
            if m in hdr:
                v = r[hdr.index(m)]
                u = units[hdr.index(m)]
                if short == "kernel":
                    v = v.split("(")[0][:48]
                parts.append(f"{short}={v}{'' if short in ('kernel','grid','regs','inst') else u}")
        print(" | ".join(parts))
        if "--stalls" in sys.argv:
            st = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                    try:
                        st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            tot = sum(x for x, _ in st) or 1
            print("    stalls: " + ", ".join(f"{n}={100*x/tot:.0f}%" for x, n in st[:6]))


if __name__ == "__main__":
    main()
