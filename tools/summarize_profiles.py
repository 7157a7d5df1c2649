"""Summarise ncu outputs of a round into profiles/ (tracked).

  python tools/summarize_profiles.py <round-tag> <launches.csv> <full.ncu-rep> [kernel-regex]

Writes profiles/<tag>_launches.md (per-kernel share of device time over the
captured launches), profiles/<tag>_<kernel>_ncu.md (key metrics of the full
capture) and profiles/traffic_k_conv.json (DRAM bytes per launch, read by
bench.py for roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"


def launches(tag, path):
    lines = [l for l in Path(path).read_text().splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        tot[name] += float(r["Metric Value"].replace(",", ""))
        cnt[name] += 1
    all_ns = sum(tot.values())
    out = [f"# {tag}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
           f"source: `{Path(path).name}` ({sum(cnt.values())} launches; cold-cache, serialised — compare shares)", "",
           "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"| {k} | {cnt[k]} | {tot[k] / 1e3:.1f} | {tot[k] / cnt[k] / 1e3:.1f} | {100 * tot[k] / all_ns:.1f}% |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(out) + "\n")
    return tot, cnt


def full(tag, rep, kernel):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
            "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
            "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
            "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
    out = [f"# {tag}: ncu --set full capture of `{kernel}`", "", f"source: `{Path(rep).name}`", "",
           "| metric | value | unit |", "|---|---|---|"]
    traffic = None
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if kernel not in d.get("Kernel Name", ""):
            continue
        u = dict(zip(hdr, units))
        for m in want:
            if m in d:
                out.append(f"| {m} | {d[m]} | {u.get(m, '')} |")
        def val(m):
            v = float(d[m].replace(",", ""))
            unit = u.get(m, "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return v * scale
        traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        inst = val("smsp__inst_executed.sum") if "smsp__inst_executed.sum" in d else None
        # pipe utilisation (FP32 FMA, XU/SFU, FP64, ALU, LSU...): % of peak over active cycles
        pipes = {}
        for m in hdr:
            if m.startswith("sm__pipe_") and m.endswith("cycles_active.avg.pct_of_peak_sustained_active") \
                    and d.get(m) not in (None, "", "n/a"):
                pipes[m[len("sm__pipe_"):-len("_cycles_active.avg.pct_of_peak_sustained_active")]] = float(d[m])
            if m.startswith("sm__inst_executed_pipe_") and m.endswith("avg.pct_of_peak_sustained_active") \
                    and d.get(m) not in (None, "", "n/a"):
                pipes["inst_" + m[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")]] = \
                    float(d[m])
        if pipes:
            out += ["", "pipe utilisation (% of peak, active cycles):", "",
                    "| pipe | % |", "|---|---|"] + [f"| {k} | {v:.1f} |" for k, v in sorted(pipes.items())]
        break
    (PROF / f"{tag}_{kernel}_ncu.md").write_text("\n".join(out) + "\n")
    return traffic, inst, pipes


if __name__ == "__main__":
    # python tools/summarize_profiles.py <tag> <launches.csv> <rep>:<kernel>[,<kernel>...] [...]
    tag, lcsv = sys.argv[1:3]
    PROF.mkdir(exist_ok=True)
    tot, cnt = launches(tag, lcsv)
    print((PROF / f"{tag}_launches.md").read_text())
    for spec in sys.argv[3:]:
        rep, kernels = spec.split(":")
        for kernel in kernels.split(","):
            traffic, inst, pipes = full(tag, rep, kernel)
            (PROF / f"traffic_{kernel}.json").write_text(json.dumps(
                {"kernel": kernel, "dram_bytes_per_launch": traffic, "warp_inst_per_launch": inst, "pipes": pipes,
                 "source": f"{tag} ncu --set full",
                 "note": ("one launch = one 960 x 6000 sigproc batch" if kernel == "k_sigproc"
                          else "one launch = one MicroBooNE event (3 planes)")}, indent=1) + "\n")
            print((PROF / f"{tag}_{kernel}_ncu.md").read_text())
