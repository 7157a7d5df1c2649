"""Workspace overflows never yield a truncated result.

The direct path's fixed-capacity tile lists (and the CSR lists, and the
profile pool) are sized by estimate; a localized shower can overflow them.
The device records the size it needed, the host entry points re-run with it
(on the same kernel, the lists grown to the real counts), and the asynchronous _device path
reports WS_ERANGE at synchronize. Each test starts from a FRESH context so
no earlier test has grown its workspace. The reference never truncates
(scatter.cpp:27-36): every frame here matches the oracle."""
import numpy as np
import pytest

from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, SimConfig, WsError, simulate_event, \
    simulate_events
from paper_2104_08265_b200.workloads import line_tracks

from .helpers import oracle_grid, oracle_response, relL2_per_channel

pytestmark = pytest.mark.gpu

GRID = GridSpec(n_wires=240, n_ticks=3000, pad_wires=20, pad_ticks=100, pitch=5.0, tick=0.5)
RESP = ResponseParams(plane_kind="collection", wire_weights=(0.1, 1.0, 0.1))
CFG = SimConfig(grid=GRID, response=RESP, fluctuate=False)


def shower(n_core=24_000, n_bg=2_000, seed=5):
    """A localized shower: n_core depos within ~2 wires and ~300 ticks (one
    8-row x 2048-tick tile gets > 20k entries), plus a sparse track
    background so the plane-average load stays light (AUTO picks direct)."""
    rng = np.random.default_rng(seed)
    bg = line_tracks(n_bg, GRID, seed=seed)
    core = line_tracks(n_core, GRID, seed=seed + 1)
    core["x"] = 600.0 + rng.uniform(0.0, 8.0, size=n_core)    # wires ~140-141 of the padded grid
    core["t"] = 500.0 + rng.uniform(0.0, 150.0, size=n_core)  # ticks ~1100-1400
    core["sigma_x"] = rng.uniform(2.5, 3.5, size=n_core)
    d = np.concatenate([bg, core])
    d["id"] = np.arange(len(d))
    return d


@pytest.fixture(scope="module")
def reference(oracle):
    d = shower()
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(GRID), d)
    return d, oracle.convolve(oracle_grid(GRID), oracle_response(RESP), s_ref)


@pytest.mark.parametrize("path", ["auto", "direct"])
def test_shower_plane_fresh_context(reference, path):
    d, m_ref = reference
    ctx = Context(0)
    ctx.set_conv_path(path)
    res = Plane(ctx, GRID, RESP).simulate(d, CFG)
    assert relL2_per_channel(res.frame, m_ref) < 1e-5
    if path == "auto":
        assert res.timing["direct_planes"] == 1  # re-run on the same (time-domain) kernel, lists grown
    ctx.close()


def test_shower_event_fresh_context(reference):
    d, m_ref = reference
    ctx = Context(0)
    ctx.set_conv_path("direct")
    planes = [Plane(ctx, GRID, RESP), Plane(ctx, GRID, RESP)]
    light = line_tracks(500, GRID, seed=9)
    frames, _ = simulate_event(ctx, planes, [light, d], CFG)
    assert relL2_per_channel(frames[1], m_ref) < 1e-5
    np.testing.assert_array_equal(frames[0], planes[0].simulate(light, CFG).frame)
    ctx.close()


SMALL = GridSpec(n_wires=64, n_ticks=1200, pad_wires=10, pad_ticks=100, pitch=5.0, tick=0.5)


def test_shower_in_long_batch_fresh_context(oracle):
    """ws_simulate_events over 300 events (more than the 256-slot header ring:
    a mid-batch drain), showers in the middle, just before the drain and at
    the end: each overflowing event is re-run, every frame is right."""
    rng = np.random.default_rng(3)
    sh = line_tracks(24_000, SMALL, seed=8)
    sh["x"] = 150.0 + rng.uniform(0.0, 8.0, size=len(sh))
    sh["t"] = 200.0 + rng.uniform(0.0, 100.0, size=len(sh))
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(SMALL), sh)
    m_ref = oracle.convolve(oracle_grid(SMALL), oracle_response(RESP), s_ref)
    ctx = Context(0)
    ctx.set_conv_path("direct")
    plane = Plane(ctx, SMALL, RESP)
    cfg = SimConfig(grid=SMALL, response=RESP, fluctuate=False)
    events = [[line_tracks(100, SMALL, seed=100 + e)] for e in range(300)]
    for e in (33, 255, 299):
        events[e] = [sh]
    out, _ = simulate_events(ctx, [plane], events, cfg)
    for e in (33, 255, 299):
        assert relL2_per_channel(out[e][0], m_ref) < 1e-5, e
    for e in (0, 32, 34, 254, 256, 298):
        np.testing.assert_array_equal(out[e][0], plane.simulate(events[e][0], cfg).frame)
    ctx.close()


def test_device_path_reports_overflow_then_fits(reference):
    """The asynchronous path: WS_ERANGE at synchronize (sized from what the
    device recorded), then the same call fits and matches."""
    import torch
    d, m_ref = reference
    ctx = Context(0)
    ctx.set_conv_path("direct")
    plane = Plane(ctx, GRID, RESP)
    dd = torch.from_numpy(d.view(np.uint8).copy()).cuda()
    fr = torch.empty(plane.shape, dtype=torch.float32, device="cuda")
    plane.simulate_device(dd, len(d), CFG, fr)
    with pytest.raises(WsError) as e:
        ctx.synchronize()
    assert e.value.code == 2 and "tile list overflow" in str(e.value)
    plane.simulate_device(dd, len(d), CFG, fr)
    ctx.synchronize()
    assert relL2_per_channel(fr.cpu().numpy(), m_ref) < 1e-5
    ctx.close()


def test_empty_call_after_direct_call_no_stale_tiles():
    """A zero-depo call behind a direct call (its k_direct must not
    start before the previous one consumed the tile counts): an empty frame."""
    import torch
    ctx = Context(0)
    ctx.set_conv_path("direct")
    plane = Plane(ctx, GRID, RESP)
    d = line_tracks(3000, GRID, seed=4)
    dd = torch.from_numpy(d.view(np.uint8).copy()).cuda()
    fr = torch.empty(plane.shape, dtype=torch.float32, device="cuda")
    fr0 = torch.full(plane.shape, 7.0, dtype=torch.float32, device="cuda")
    for _ in range(5):
        plane.simulate_device(dd, len(d), CFG, fr)
        plane.simulate_device(dd, 0, CFG, fr0)
    ctx.synchronize()
    assert float(fr0.abs().max()) == 0.0
    ctx.close()


def _fluct_u32(grid, resp, d, seed):
    import torch
    from paper_2104_08265_b200 import RngConfig
    cfg = SimConfig(grid=grid, response=resp, fluctuate=True, rng=RngConfig(mode="philox", seed=seed))
    ctx = Context(0)
    plane = Plane(ctx, grid, resp)
    dd = torch.from_numpy(d.view(np.uint8).copy()).cuda()
    ch = torch.empty(plane.shape, dtype=torch.int32, device="cuda")
    fr = torch.empty(plane.shape, dtype=torch.float32, device="cuda")
    plane.simulate_device(dd, len(d), cfg, fr, ch, charge_type="u32")
    ctx.synchronize()
    out = ch.cpu().numpy().view(np.uint32).astype(np.int64), fr.cpu().numpy()
    ctx.close()
    return out


def test_fluctuation_high_charge_exact(oracle):
    """Integer charge grid (u32 atomics): cells far beyond 2^24 electrons,
    summed over many stacked depos, stay exact (the reference's grid is
    int64, core.hpp:94-99; the old fp32 grid was exact only below 2^24)."""
    grid = GridSpec(n_wires=40, n_ticks=400, pad_wires=10, pad_ticks=100)
    resp = ResponseParams()
    rng = np.random.default_rng(8)
    d = line_tracks(400, grid, seed=3)
    d["x"] = 100.0 + rng.uniform(0.0, 0.5, size=len(d))  # all stacked on ~5 wires x ~10 ticks
    d["t"] = 100.0 + rng.uniform(0.0, 0.5, size=len(d))
    d["q"] = 2_000_000
    s_ref, _ = oracle.charge_fluct_on(oracle_grid(grid), d, rng_mode=1, seed=3)
    assert s_ref.max() > 2 ** 25
    s, m = _fluct_u32(grid, resp, d, 3)
    np.testing.assert_array_equal(s, s_ref)
    m_ref = oracle.convolve(oracle_grid(grid), oracle_response(resp), s_ref.astype(np.float64))
    assert relL2_per_channel(m, m_ref) < 1e-5


def test_fluctuation_extreme_depo_charge(oracle):
    """2e8 electrons per depo: the walk's pmf seed goes through lgamma(n + 1)
    ~ 4e9, where CUDA's and glibc's lgamma differ by ulps (~1e-6 absolute in
    the exponent), which can move a rare draw by a few electrons. Charge is
    conserved exactly per depo (the remainder rule), the grid stays within a
    few electrons, the frame within the tolerance."""
    grid = GridSpec(n_wires=40, n_ticks=400, pad_wires=10, pad_ticks=100)
    resp = ResponseParams()
    d = line_tracks(60, grid, seed=3)
    d["q"] = np.int64(200_000_000)
    s_ref, _ = oracle.charge_fluct_on(oracle_grid(grid), d, rng_mode=1, seed=3)
    s, m = _fluct_u32(grid, resp, d, 3)
    assert s.sum() == s_ref.sum()
    diff = np.abs(s - s_ref)
    assert diff.max() <= 16 and (diff > 0).mean() < 1e-3
    m_ref = oracle.convolve(oracle_grid(grid), oracle_response(resp), s_ref.astype(np.float64))
    assert relL2_per_channel(m, m_ref) < 1e-5


def test_fluctuation_charge_types_past_2_32():
    """The count grid is u64 (the reference's is int64): 4 delta depos of 3e10
    electrons on one cell sum exactly; the int64 charge output carries it,
    the uint32 output is an error (never a wrapped count)."""
    import torch
    from paper_2104_08265_b200 import RngConfig
    grid = GridSpec(n_wires=20, n_ticks=300, pad_wires=10, pad_ticks=100)
    resp = ResponseParams()
    d = line_tracks(4, grid, seed=3)
    d["q"] = np.int64(30_000_000_000)
    d["sigma_t"] = 0.0
    d["sigma_x"] = 0.0
    d["x"], d["t"] = 50.0, 75.0  # one cell takes all 1.2e11 electrons
    cfg = SimConfig(grid=grid, response=resp, fluctuate=True, rng=RngConfig(mode="philox"))
    ctx = Context(0)
    plane = Plane(ctx, grid, resp)
    dd = torch.from_numpy(d.view(np.uint8).copy()).cuda()
    fr = torch.empty(plane.shape, dtype=torch.float32, device="cuda")
    ch64 = torch.zeros(plane.shape, dtype=torch.int64, device="cuda")
    plane.simulate_device(dd, len(d), cfg, fr, ch64, charge_type="i64")
    ctx.synchronize()
    c = ch64.cpu().numpy()
    assert c.max() == 120_000_000_000 and c.sum() == 120_000_000_000
    ch32 = torch.zeros(plane.shape, dtype=torch.int32, device="cuda")
    plane.simulate_device(dd, len(d), cfg, fr, ch32, charge_type="u32")
    with pytest.raises(WsError) as e:
        ctx.synchronize()
    assert e.value.code == 4 and "4294967295" in str(e.value)
    ctx.close()
