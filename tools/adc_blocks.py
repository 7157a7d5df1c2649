import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2104_08265_b200 import AdcConfig, Context, Plane, SimConfig, RngConfig, run_events
from paper_2104_08265_b200.workloads import microboone_event, microboone_grids
ctx = Context(0)
grids, resps = microboone_grids()
planes = [Plane(ctx, g, r) for g, r in zip(grids, resps)]
ev = microboone_event(100_000, seed=1)
cfg = SimConfig(fluctuate=False, rng=RngConfig(mode="philox", seed=12345), adc=AdcConfig(1.0, 2048.0, 12))
adcs = [[np.empty(p.shape, dtype=np.uint16) for p in planes]]
run_events(ctx, planes, [ev], cfg, adc_type="u16", adcs=adcs)
for B in (32, 64, 128):
    tot = const = byte = nib = 0
    for a in adcs[0]:
        W, N = a.shape
        nb = N // B
        x = a[:, :nb * B].reshape(W, nb, B).astype(np.int32)
        rng_ = x.max(-1) - x.min(-1)
        tot += rng_.size; const += (rng_ == 0).sum(); nib += ((rng_ > 0) & (rng_ < 16)).sum(); byte += ((rng_ >= 16) & (rng_ < 256)).sum()
    raw = tot - const - byte - nib
    comp = (tot * 4 + (nib * B // 2) + byte * B + raw * B * 2)
    print(f"B={B}: blocks {tot} const {const/tot:.3f} nib {nib/tot:.3f} byte {byte/tot:.3f} raw {raw/tot:.3f}  bytes {comp/1e6:.1f} MB vs {sum(a.nbytes for a in adcs[0])/1e6:.1f}")
