import numpy as np, torch
from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, SimConfig
from paper_2104_08265_b200.workloads import line_tracks
GRID = GridSpec(n_wires=240, n_ticks=3000, pad_wires=20, pad_ticks=100, pitch=5.0, tick=0.5)
RESP = ResponseParams(plane_kind="collection", wire_weights=(0.1, 1.0, 0.1))
CFG = SimConfig(grid=GRID, response=RESP, fluctuate=False)
ctx = Context(0); ctx.set_conv_path("direct")
plane = Plane(ctx, GRID, RESP)
d = line_tracks(3000, GRID, seed=4)
dd = torch.from_numpy(d.view(np.uint8).copy()).cuda()
fr = torch.empty(plane.shape, dtype=torch.float32, device="cuda")
fr0 = torch.full(plane.shape, 7.0, dtype=torch.float32, device="cuda")
for i in range(3):
    plane.simulate_device(dd, len(d), CFG, fr); print("ok a", i, flush=True)
    plane.simulate_device(dd, 0, CFG, fr0); print("ok b", i, flush=True)
ctx.synchronize(); print("max", float(fr0.abs().max()))
