"""Integer charge-grid differences GPU vs oracle for the test_skip_records
workloads (diagnostics: which units / bins differ and by how much)."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from oracle.oracle import Oracle
from paper_2104_08265_b200 import Context
from paper_2104_08265_b200.workloads import line_tracks
from tests.test_gpu_fluct_walk import GRID, _charge
from tests.helpers import oracle_grid

shape = sys.argv[1] if len(sys.argv) > 1 else "huge_q"
rng_mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(17)
d = line_tracks(1500, GRID, seed=13)
if shape == "huge_q":
    d["q"] = rng.integers(200_000, 900_000, size=len(d))
s_ref, _ = Oracle().charge_fluct_on(oracle_grid(GRID), d, rng_mode=rng_mode, seed=31)
ctx = Context(0)
s = _charge(ctx, d, rng_mode, 31).astype(np.int64)
ctx.close()
diff = s - s_ref
nz = np.argwhere(diff != 0)
print(shape, rng_mode, "cells differing", len(nz), "max |diff|", np.abs(diff).max(), "sum diff", diff.sum(), "total", s_ref.sum())
for w, t in nz[:10]:
    print("  cell", w, t, "gpu", s[w, t], "ref", s_ref[w, t])
