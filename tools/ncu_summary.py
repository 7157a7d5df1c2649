"""Key ncu metrics per kernel from a .ncu-rep (raw page)."""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
STALL = "smsp__average_warps_issue_stalled_"


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("==", d["Kernel Name"][:80])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]} {units[hdr.index(k)]}")
        st = sorted(((float(d[k]), k[len(STALL):]) for k in hdr if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")
                     and d[k] not in ("", "n/a")), reverse=True)[:6]
        print("  stalls/issue:", ", ".join(f"{n.replace('_per_issue_active.ratio','')}={v:.2f}" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
