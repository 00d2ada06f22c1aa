"""Summarize an ncu report (--page raw --csv) into a markdown table of the metrics the
roofline discussion uses.  Usage: python scripts/ncu_summary.py report.ncu-rep > out.md"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem thru %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "fp64 tensor ops % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(path, header=True):
    if path.endswith(".csv"):  # a raw page exported on the GPU box (profile_round.sh)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
    if header:
        print("| kernel | " + " | ".join(m[1] for m in METRICS) + " | top stalls |")
        print("|---" * (len(METRICS) + 2) + "|")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")[-48:]
        cells = []
        for m, _ in METRICS:
            if m in hdr:
                i = hdr.index(m)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        vals = [(float(r[i].replace(",", "") or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")) for i in stall_cols]
        tot = sum(v for v, _ in vals) or 1.0
        top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(vals, reverse=True)[:3])
        print(f"| {name} | " + " | ".join(cells) + f" | {top} |")


if __name__ == "__main__":
    for i, p in enumerate(sys.argv[1:]):
        main(p, header=i == 0)
