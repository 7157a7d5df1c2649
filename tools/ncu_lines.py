"""Summarise an ncu source page (cuda,sass CSV) by CUDA source line: stall samples and instructions."""
import csv, sys, subprocess

def main(rep, kernel, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    path, hdr, agg = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0] not in ("", "Function Name"):
            d = dict(zip(hdr, r))
            try:
                agg.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"]), path, r[0], r[1][:90]))
            except (ValueError, KeyError):
                pass
    tot_s = sum(a[0] for a in agg) or 1
    tot_i = sum(a[1] for a in agg) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for s, i, p, ln, src in sorted(agg, reverse=True)[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {p}:{ln}  {src}")

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
