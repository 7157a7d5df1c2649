import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2104_08265_b200 import *
from paper_2104_08265_b200._lib import WsError
from oracle.oracle import Oracle
from tests.helpers import oracle_grid
o = Oracle()
ctx = Context(0)
grid = GridSpec(n_wires=480, n_ticks=6000)
depos = gen_depos(2000, 7, grid)
for mode in (0, 1):
    cfg = SimConfig(grid=grid, fluctuate=True, rng=RngConfig(mode="philox" if mode else "substream"))
    res = Plane(ctx, grid, ResponseParams()).simulate(depos, cfg, want_charge=True)
    s_ref, _ = o.charge_fluct_on(oracle_grid(grid), depos, rng_mode=mode, seed=12345)
    g = res.charge.astype(np.int64)
    print('mode', mode, 'sum gpu', g.sum(), 'ref', s_ref.sum(), 'ndiff', (g != s_ref).sum(), res.timing)
    for i in range(3):
        d = depos[i:i+1]
        r1 = Plane(ctx, grid, ResponseParams()).simulate(d, cfg, want_charge=True).charge.astype(np.int64)
        s1, _ = o.charge_fluct_on(oracle_grid(grid), d, rng_mode=mode, seed=12345)
        nz = np.nonzero(s1)
        print(' depo', i, 'q', d['q'][0], 'gpu sum', r1.sum(), 'ref sum', s1.sum(), 'ndiff', (r1 != s1).sum())
        print('   ref', s1[nz][:12]); print('   gpu', r1[nz][:12])
# drift
dp2 = DriftParams(response_plane_x=100.0, enabled=True)
try:
    r = Plane(ctx, grid, ResponseParams()).simulate(depos, SimConfig(grid=grid, fluctuate=False, drift=dp2))
    print('no error raised', r.timing)
except WsError as e:
    print('raised', e)
