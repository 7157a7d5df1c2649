"""Quick device timing of the sigproc chain (960 x 6000 by default)."""
import sys
import numpy as np
import torch
from paper_2104_08265_b200 import Context, sigproc_chain, sigproc_chain_device

rows, cols = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (960, 6000)
ctx = Context(0)
rng = np.random.default_rng(1)
data = rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))
filt = rng.normal(size=cols) + 1j * rng.normal(size=cols)
dd, fd = torch.from_numpy(data).cuda(), torch.from_numpy(filt).cuda()
blk = torch.empty((rows - 80, cols), dtype=torch.float64, device="cuda")
med = torch.empty(rows - 80, dtype=torch.float64, device="cuda")
stream = torch.cuda.ExternalStream(ctx.stream)
for want_med in (True, False):
    for _ in range(3):
        sigproc_chain_device(ctx, dd, rows, cols, fd, blk, med if want_med else None, pad_rows=80)
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record(stream)
    for _ in range(K):
        sigproc_chain_device(ctx, dd, rows, cols, fd, blk, med if want_med else None, pad_rows=80)
    e1.record(stream)
    e1.synchronize()
    us = e0.elapsed_time(e1) / K * 1e3
    nbytes = rows * cols * 16 + (rows - 80) * cols * 8
    print(f"medians={want_med}: {us:.1f} us/chain  {nbytes / us / 1e3:.0f} GB/s algorithmic")
pin = torch.from_numpy(data).pin_memory().numpy()
import time
for _ in range(2):
    sigproc_chain(pin, filt, 80, ctx=ctx)
t = time.perf_counter()
for _ in range(5):
    sigproc_chain(pin, filt, 80, ctx=ctx)
print(f"host path (pinned in, pageable out): {(time.perf_counter() - t) / 5 * 1e3:.2f} ms/chain")
