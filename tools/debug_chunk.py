import numpy as np, sys
sys.path.insert(0, '.')
from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, SimConfig
from paper_2104_08265_b200.workloads import line_tracks
from oracle.oracle import Oracle
from tests.helpers import oracle_grid, oracle_response, relL2_per_channel
ctx = Context(0); o = Oracle()
grid = GridSpec(n_wires=16, n_ticks=900, pad_wires=10, pad_ticks=100, pitch=5.0, tick=0.5)
resp = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))
for nd in (2000, 6000, 7000, 8000, 12000):
    d = line_tracks(nd, grid, seed=12)
    d["x"] = 40.0 + (d["x"] % 3.0)
    d["sigma_x"] = 2.5
    s_ref, _ = o.charge_fluct_off(oracle_grid(grid), d)
    m_ref = o.convolve(oracle_grid(grid), oracle_response(resp), s_ref)
    out = []
    for path in ("direct", "fft"):
        ctx.set_conv_path(path)
        m = Plane(ctx, grid, resp).simulate(d, SimConfig(grid=grid, response=resp, fluctuate=False)).frame
        num = np.sqrt(((m - m_ref) ** 2).sum(1)); den = np.sqrt((m_ref ** 2).sum(1))
        out.append((path, relL2_per_channel(m, m_ref), np.argmax(np.where(den > 0, num / np.maximum(den, 1e-300), 0))))
    print(nd, out, flush=True)
