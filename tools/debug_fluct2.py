import sys; sys.path.insert(0, '.')
import numpy as np, ctypes as C
from paper_2104_08265_b200 import *
from oracle.oracle import Oracle
from tests.helpers import oracle_grid
o = Oracle()
ctx = Context(0)
grid = GridSpec(n_wires=480, n_ticks=6000)
depos = gen_depos(2000, 7, grid)
og = oracle_grid(grid)
for mode in (1, 0):
    cfg = SimConfig(grid=grid, fluctuate=True, rng=RngConfig(mode="philox" if mode else "substream"))
    pl = Plane(ctx, grid, ResponseParams())
    bad = []
    for i in range(len(depos)):
        d = depos[i:i+1]
        r1 = pl.simulate(d, cfg, want_charge=True).charge.astype(np.int64)
        s1, _ = o.charge_fluct_on(og, d, rng_mode=mode, seed=12345)
        if (r1 != s1).any():
            bad.append(i)
            p = o.sample_patch(og, d)
            vals = p['values'].ravel()
            nz = np.nonzero((r1 != s1).ravel())[0]
            print('mode', mode, 'depo', i, d, 'n bins', vals.size)
            rr = r1[p['wire_offset']:p['wire_offset']+p['n_w'], p['tick_offset']:p['tick_offset']+p['n_t']].ravel()
            ss = s1[p['wire_offset']:p['wire_offset']+p['n_w'], p['tick_offset']:p['tick_offset']+p['n_t']].ravel()
            first = np.nonzero(rr != ss)[0][0]
            rem = d['q'][0] - ss[:first].sum()
            prem = 1.0 - vals[:first].sum()
            print('  first diff bin', first, 'gpu', rr[first], 'ref', ss[first], 'remaining~', rem, 'p~', vals[first]/prem)
    print('mode', mode, 'bad depos', bad)
