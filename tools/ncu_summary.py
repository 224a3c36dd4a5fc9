"""One-kernel summary of an ncu --set full report (for profiles/).

usage: python tools/ncu_summary.py REPORT.ncu-rep "title line" > profiles/rNN_....txt
"""
import csv
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_imma.sum",
    "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]


def main():
    rep, title = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units = r[0], r[1]
    print(title)
    for v in r[2:]:
        for k in KEYS:
            if k in h and v[h.index(k)] not in ("", "n/a"):
                i = h.index(k)
                print("%-64s %s %s" % (k, v[i], units[i]))
        print()
    stalls = {}
    for i, k in enumerate(h):
        p = "smsp__pcsamp_warps_issue_stalled_"
        if k.startswith(p) and not k.endswith("not_issued"):
            try:
                stalls[k[len(p):]] = int(float(v[i] or 0))
            except ValueError:
                pass
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
    print("top stall samples: " + ", ".join("%s=%d" % kv for kv in top))


if __name__ == "__main__":
    main()
