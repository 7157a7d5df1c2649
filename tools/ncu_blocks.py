"""Hottest straight-line SASS runs (instructions executed) of one kernel in an ncu report."""
import csv, subprocess, sys

def main(rep, kernel, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout
    hdr, runs = None, []
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            c = int(d["Instructions Executed"] or 0)
            src = d["Source"].strip()
            if runs and runs[-1][0] == c:
                runs[-1][1] += 1
                runs[-1][3] = src
            else:
                runs.append([c, 1, src, src])
    tot = sum(c * n for c, n, _, _ in runs) or 1
    print(f"total warp instructions {tot}")
    for c, n, a, b in sorted(runs, key=lambda x: -x[0] * x[1])[:top]:
        print(f"{100*c*n/tot:5.1f}%  {c:>9} x {n:3d}  {a[:45]:45s} .. {b[:45]}")

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
