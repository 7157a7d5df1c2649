"""Per-channel relL2 of both convolution kernels vs the oracle on a few
configurations (GPU; diagnostic, prints a table)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, SimConfig
from paper_2104_08265_b200.workloads import line_tracks, microboone_event, microboone_grids
from oracle.oracle import Oracle
from tests.helpers import oracle_grid, oracle_response, relL2_per_channel

ctx = Context(0)
o = Oracle()
cases = []
g = GridSpec(n_wires=64, n_ticks=800, pad_wires=20, pad_ticks=100)
cases.append(("smoke induction 3-tap", g, ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1)),
              line_tracks(400, g, seed=7)))
g = GridSpec(n_wires=480, n_ticks=6000)
cases.append(("C1 collection", g, ResponseParams(), line_tracks(10_000, g, seed=1)))
cases.append(("C1 induction", g, ResponseParams(plane_kind="induction"), line_tracks(10_000, g, seed=1)))
grids, resps = microboone_grids()
ev = microboone_event(100_000, seed=1)
cases.append(("MicroBooNE U (induction)", grids[0], resps[0], ev[0]))
cases.append(("MicroBooNE W (collection)", grids[2], resps[2], ev[2]))
for name, grid, resp, d in cases:
    s_ref, _ = o.charge_fluct_off(oracle_grid(grid), d)
    m_ref = o.convolve(oracle_grid(grid), oracle_response(resp), s_ref)
    row = [name]
    for path in ("direct", "fft"):
        ctx.set_conv_path(path)
        m = Plane(ctx, grid, resp).simulate(d, SimConfig(grid=grid, response=resp, fluctuate=False)).frame
        row.append(f"{path} {relL2_per_channel(m, m_ref):.2e}")
    print(" | ".join(row), flush=True)
