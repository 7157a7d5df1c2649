"""Quick device-time probe of one MicroBooNE-scale event (development aid)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2104_08265_b200 import Context, Plane, SimConfig, simulate_event_device
from paper_2104_08265_b200._lib import TimingC
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids

ctx = Context(0)
grids, resps = microboone_grids()
planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
print([p.info for p in planes])
depos = microboone_event(100_000, seed=1)
dd = [torch.from_numpy(d.view(np.uint8)).cuda() for d in depos]
frames = [torch.empty(p.shape, dtype=torch.float32, device='cuda') for p in planes]
fluct = len(sys.argv) > 1 and sys.argv[1] == 'on'
cfg = SimConfig(fluctuate=fluct)
torch.cuda.synchronize()
for it in range(6):
    t = TimingC()
    simulate_event_device(ctx, planes, dd, [len(d) for d in depos], cfg, frames, timing=t)
    ctx.synchronize()
    print(it, {k: round(v, 4) if isinstance(v, float) else v for k, v in t.as_dict().items()})
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(ctx.stream)
n = 20
s.record(st)
for it in range(n):
    simulate_event_device(ctx, planes, dd, [len(d) for d in depos], cfg, frames)
e.record(st)
ctx.synchronize(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
print(f"event {ms:.3f} ms  -> {1e5/ms*1e3:.3e} depos/s, {1e3/ms:.1f} events/s; launches={ctx.launch_count}")
