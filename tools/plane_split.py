"""C2 event: one 3-plane call (simulate_event_device) vs three plane calls
(simulate_device per plane: each plane's profiles are still in L2 when its
k_direct reads them), device time per event over rotating events."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2104_08265_b200 import Context, Plane, SimConfig, simulate_event_device
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids

ctx = Context(0)
grids, resps = microboone_grids()
planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
evs = [microboone_event(100_000, seed=s) for s in range(1, 5)]
dev = [[torch.from_numpy(d.view(np.uint8)).cuda() for d in ev] for ev in evs]
n = [[len(d) for d in ev] for ev in evs]
frames = [torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes]
cfg = SimConfig(fluctuate=False)
s = torch.cuda.current_stream()


def one(i):
    simulate_event_device(ctx, planes, dev[i % 4], n[i % 4], cfg, frames)


def split(i):
    for k, p in enumerate(planes):
        p.simulate_device(dev[i % 4][k], n[i % 4][k], cfg, frames[k])


for name, fn in (("event", one), ("planes", split), ("event", one), ("planes", split)):
    for i in range(5):
        fn(i)
    ctx.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    # the library runs on its own stream: bracket with synchronizes and wall-clock events on it
    import time
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for i in range(40):
        fn(i)
    ctx.synchronize()
    w1 = time.perf_counter()
    print(f"{name:7s} {(w1 - w0) / 40 * 1e3:.4f} ms/event (wall, 40 events)")
