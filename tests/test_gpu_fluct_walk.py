"""The two-pass exact walk (k_fluct_prep -> k_fluct_walk, ws_sample.cu) and
its fallbacks, against the oracle's integer charge grid (fluctuate +
binomial, rasterize.cpp:124-157, rng.cpp:146-193):

* units whose draws could take binomial's normal branch (q min(p, 1-p) >
  1e6, rng.cpp:181-186) go whole to the one-pass walk, mixed in one call
  with record-walked units;
* a fresh context whose record capacity (160 per unit) is too small for wide
  depos re-runs the call with the recorded need (never a partial grid);
* both RNG streams; delta depos (one bin: no draw at all);
* skip records (runs of draws that take 0 electrons for any n <= q) across
  wire rows, at a unit's end, whole units of them, and almost none.
"""
import numpy as np
import pytest

from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, RngConfig, SimConfig
from paper_2104_08265_b200.workloads import line_tracks

from .helpers import oracle_grid

pytestmark = pytest.mark.gpu

GRID = GridSpec(n_wires=200, n_ticks=1200, pad_wires=20, pad_ticks=100, pitch=5.0, tick=0.5)


def _charge(ctx, depos, rng_mode, seed):
    resp = ResponseParams()
    cfg = SimConfig(grid=GRID, response=resp, fluctuate=True,
                    rng=RngConfig(mode="philox" if rng_mode else "substream", seed=seed))
    return Plane(ctx, GRID, resp).simulate(depos, cfg, want_charge=True).charge


@pytest.mark.parametrize("rng_mode", [0, 1])
def test_mixed_record_and_normal_branch_units(oracle, rng_mode):
    rng = np.random.default_rng(11)
    d = line_tracks(3000, GRID, seed=5)
    big = rng.random(len(d)) < 0.03
    d["q"][big] = 4_000_000  # p ~ 0.5 bins: q min(p, 1 - p) > 1e6 -> normal branch possible
    d["sigma_t"][:5] = 0.0   # delta depos: a single bin, no draw
    d["sigma_x"][:5] = 0.0
    s_ref, _ = oracle.charge_fluct_on(oracle_grid(GRID), d, rng_mode=rng_mode, seed=21)
    assert s_ref.max() < 2 ** 24
    ctx = Context(0)
    try:
        s = _charge(ctx, d, rng_mode, 21)
    finally:
        ctx.close()
    np.testing.assert_array_equal(s.astype(np.int64), s_ref)


def test_record_overflow_reruns_on_fresh_context(oracle):
    """Wide depos: ~60 x 50 bins each, far above the initial 160 records per
    unit; the host call re-runs with the recorded need and the grid is exact."""
    d = line_tracks(400, GRID, seed=9)
    d["sigma_t"] = 4.0   # us: +-3 sigma over ~50 ticks
    d["sigma_x"] = 40.0  # mm: ~50 wires
    s_ref, _ = oracle.charge_fluct_on(oracle_grid(GRID), d, rng_mode=1, seed=4)
    ctx = Context(0)
    try:
        s = _charge(ctx, d, 1, 4)
        s2 = _charge(ctx, d, 1, 4)  # the grown workspace: one pass
    finally:
        ctx.close()
    np.testing.assert_array_equal(s.astype(np.int64), s_ref)
    np.testing.assert_array_equal(s2, s)


@pytest.mark.parametrize("rng_mode", [0, 1])
@pytest.mark.parametrize("shape", ["tails", "one_tick", "one_wire", "tiny_q", "huge_q"])
def test_skip_records(oracle, rng_mode, shape):
    """Runs of certain-zero draws (p = 0, or q log1p(-pp) > log u + 4e-5)
    are one skip record that k_fluct_walk crosses in one step: runs that span
    wire rows (one tick per row: a row wrap at every bin), runs that reach the
    unit's last record, units made of skips only (q = 1..3), and units with
    almost none (q ~ 1e5 per bin). The integer grid is the oracle's."""
    rng = np.random.default_rng(17)
    d = line_tracks(1500, GRID, seed=13)
    if shape == "tails":
        d["sigma_t"] = rng.uniform(1.5, 3.0, size=len(d))   # long Gaussian tails in ticks and wires
        d["sigma_x"] = rng.uniform(8.0, 15.0, size=len(d))
        d["q"] = rng.integers(50, 5000, size=len(d))
    elif shape == "one_tick":
        d["sigma_t"] = 0.0                                   # n_t = 1: every bin ends a wire row
        d["sigma_x"] = rng.uniform(5.0, 20.0, size=len(d))
    elif shape == "one_wire":
        d["sigma_x"] = 0.0                                   # n_w = 1: one row
        d["sigma_t"] = rng.uniform(0.5, 3.0, size=len(d))
    elif shape == "tiny_q":
        d["q"] = rng.integers(1, 4, size=len(d))             # nearly every draw is a certain zero
    else:
        d["q"] = rng.integers(200_000, 900_000, size=len(d))  # few certain zeros (q min(p, 1-p) stays < 1e6 mostly)
    s_ref, _ = oracle.charge_fluct_on(oracle_grid(GRID), d, rng_mode=rng_mode, seed=31)
    ctx = Context(0)
    try:
        s = _charge(ctx, d, rng_mode, 31)
    finally:
        ctx.close()
    s = s.astype(np.int64)
    np.testing.assert_array_equal(s, s_ref)
    assert s.sum() == s_ref.sum()
