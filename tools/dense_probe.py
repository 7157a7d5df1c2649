import sys, pathlib; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2104_08265_b200 import Context, Plane, SimConfig, simulate_event_device, simulate_events
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids
cfg = SimConfig(fluctuate=False)
for n in [300_000, 1_000_000]:
    ev = microboone_event(n, seed=3)
    for path in ("direct", "fft"):
        ctx = Context(0); ctx.set_conv_path(path)
        grids, resps = microboone_grids()
        planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
        outs = [[np.empty(p.shape, np.float32) for p in planes]]
        simulate_events(ctx, planes, [ev], cfg, frames=outs)
        dev = [torch.from_numpy(d.view(np.uint8)).cuda() for d in ev]
        fr = [torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes]
        nn = [len(d) for d in ev]
        for _ in range(2): simulate_event_device(ctx, planes, dev, nn, cfg, fr)
        ctx.synchronize()
        s = torch.cuda.ExternalStream(ctx.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5): simulate_event_device(ctx, planes, dev, nn, cfg, fr)
        e1.record(s); ctx.synchronize()
        print(f"{n} depos, {path}: {e0.elapsed_time(e1) / 5:.3f} ms/event", flush=True)
        ctx.close()
