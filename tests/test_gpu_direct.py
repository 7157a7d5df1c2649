"""GPU parity of the two convolution kernels (time-domain k_direct and row-FFT
k_conv) and of the per-band routing between them, against the CPU oracle
(wsoracle.c's direct circular convolution, pinned to the reference in
test_oracle.py) and against each other.

Tolerances as in test_gpu_parity.py (BASELINE.json north_star): per-channel
relative L2 <= 1e-5 on the frame."""
import numpy as np
import pytest

from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, SimConfig, simulate_event
from paper_2104_08265_b200.workloads import line_tracks, microboone_event, microboone_grids

from .helpers import oracle_grid, oracle_response, relL2_per_channel

pytestmark = pytest.mark.gpu

TOL_FRAME = 1e-5
SMALL = GridSpec(n_wires=96, n_ticks=900, pad_wires=20, pad_ticks=100, pitch=5.0, tick=0.5)


@pytest.fixture(scope="module")
def pctx():
    c = Context(0)
    yield c
    c.close()


def _frame(ctx, path, grid, resp, depos, kappa=None):
    ctx.set_conv_path(path)
    if kappa is not None:
        ctx.set_direct_kappa(kappa)
    try:
        return Plane(ctx, grid, resp).simulate(depos, SimConfig(grid=grid, response=resp, fluctuate=False)).frame
    finally:
        ctx.set_conv_path("auto")
        ctx.set_direct_kappa(128.0)


@pytest.mark.parametrize("path", ["direct", "fft", "auto"])
@pytest.mark.parametrize("kind", ["collection", "induction"])
@pytest.mark.parametrize("ww", [(1.0,), (0.1, 1.0, 0.1), (-0.05, 0.2, 1.0, 0.2, -0.05)])
def test_paths_vs_oracle_small(pctx, oracle, path, kind, ww):
    resp = ResponseParams(plane_kind=kind, wire_weights=ww)
    depos = line_tracks(600, SMALL, seed=3)
    m = _frame(pctx, path, SMALL, resp, depos)
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(SMALL), depos)
    m_ref = oracle.convolve(oracle_grid(SMALL), oracle_response(resp), s_ref)
    assert relL2_per_channel(m, m_ref) < TOL_FRAME


@pytest.mark.parametrize("shaper", [0.0, 1.0, 2.0])
def test_direct_c1_folded_and_long_kernels(pctx, oracle, shaper):
    """configs[0] geometry (padded ticks 6200, not 7-smooth: the FFT path folds
    a longer transform; the direct path is circular by construction), with
    kernels from 114 to >300 taps (several 128-tap chunks per profile)."""
    grid = GridSpec(n_wires=480, n_ticks=6000, pad_wires=100, pad_ticks=400)
    resp = ResponseParams(plane_kind="collection", shaper_peaking=shaper)
    depos = line_tracks(10_000, grid, seed=1)
    m = _frame(pctx, "direct", grid, resp, depos)
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(grid), depos)
    m_ref = oracle.convolve(oracle_grid(grid), oracle_response(resp), s_ref)
    assert relL2_per_channel(m, m_ref) < TOL_FRAME


def test_direct_wrap_both_edges(pctx, oracle):
    """Depos hugging tick 0 and the last tick: the response wraps circularly
    (the reference's convolve is circular, spectral.cpp:141-175)."""
    grid = GridSpec(n_wires=30, n_ticks=200, pad_wires=5, pad_ticks=100)
    resp = ResponseParams(plane_kind="induction", wire_weights=(0.2, 1.0, 0.2))
    d = line_tracks(40, grid, seed=2)
    d["t"][:20] = -49.5   # tick ~1 of the padded grid
    d["t"][20:] = 149.6   # last padded ticks
    d["x"][:5] = -20.0    # wire wrap across the padded edge
    m = _frame(pctx, "direct", grid, resp, d)
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(grid), d)
    m_ref = oracle.convolve(oracle_grid(grid), oracle_response(resp), s_ref)
    assert relL2_per_channel(m, m_ref) < TOL_FRAME


def test_auto_routes_per_plane_bitwise(pctx):
    """AUTO routes each plane of a call by its depo load: a sparse plane and a
    dense plane in one event take different kernels, and each frame is
    bitwise the frame of the kernel it was routed to."""
    grid = GridSpec(n_wires=400, n_ticks=2000, pad_wires=20, pad_ticks=100)
    resp = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))
    sparse = line_tracks(2_000, grid, seed=4)
    dense = line_tracks(60_000, grid, seed=5)
    planes = [Plane(pctx, grid, resp), Plane(pctx, grid, resp)]
    cfg = SimConfig(fluctuate=False)
    forced = {}
    for path in ("fft", "direct"):
        pctx.set_conv_path(path)
        forced[path] = [p.simulate(d, cfg).frame for p, d in zip(planes, (sparse, dense))]
    pctx.set_conv_path("auto")
    # work estimate per plane = depos x 12 x (n_lags + 16); cells = W x Np
    pctx.set_direct_kappa(10.0)
    try:
        frames, _ = simulate_event(pctx, planes, [sparse, dense], cfg)
    finally:
        pctx.set_direct_kappa(128.0)
    np.testing.assert_array_equal(frames[0], forced["direct"][0])
    np.testing.assert_array_equal(frames[1], forced["fft"][1])
    for i in range(2):
        assert relL2_per_channel(forced["direct"][i], forced["fft"][i]) < TOL_FRAME


def test_direct_deterministic(pctx):
    grid = SMALL
    resp = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))
    d = line_tracks(3000, grid, seed=8)
    a = _frame(pctx, "direct", grid, resp, d)
    b = _frame(pctx, "direct", grid, resp, d)
    np.testing.assert_array_equal(a, b)


def test_microboone_u_plane_full_size(pctx, oracle):
    """configs[1] at full size (the bench workload): the U plane of a 100k-depo
    event (2600 x 9800 padded) against the oracle, both kernels; and the whole
    event through the batched API equals the single planes."""
    grids, resps = microboone_grids()
    ev = microboone_event(100_000, seed=1)
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(grids[0]), ev[0])
    m_ref = oracle.convolve(oracle_grid(grids[0]), oracle_response(resps[0]), s_ref)
    for path in ("direct", "fft"):
        m = _frame(pctx, path, grids[0], resps[0], ev[0])
        assert relL2_per_channel(m, m_ref) < TOL_FRAME, path
    planes = [Plane(pctx, g, r) for g, r in zip(grids, resps)]
    frames, _ = simulate_event(pctx, planes, ev, SimConfig(fluctuate=False))
    for p, d, f in zip(planes, ev, frames):
        np.testing.assert_array_equal(p.simulate(d, SimConfig(fluctuate=False)).frame, f)


def test_direct_band_beyond_staging(oracle):
    """A band with more depos than k_direct stages at once (chunked
    accumulation) still matches the oracle. A fresh context: the tile list
    capacity starts at its default, so the ~12k-entry tiles overflow it and
    the host re-runs with the recorded size (never a truncated tile)."""
    pctx = Context(0)
    grid = GridSpec(n_wires=16, n_ticks=900, pad_wires=10, pad_ticks=100, pitch=5.0, tick=0.5)
    # unipolar response: 12k stacked bipolar responses cancel to ~1e-3 of
    # their absolute sum, which any fp32 method resolves only to ~1e-6
    resp = ResponseParams(plane_kind="collection", wire_weights=(0.1, 1.0, 0.1))
    d = line_tracks(12_000, grid, seed=12)
    # every depo centred on wire 18 of the padded grid; sigma_x keeps the
    # footprint's edge wires well-conditioned (a 10-sigma tail bin is fp64
    # erf rounding noise, where CUDA's and glibc's erf legitimately differ)
    d["x"] = 40.0 + (d["x"] % 3.0)
    d["sigma_x"] = 2.5
    m = _frame(pctx, "direct", grid, resp, d)
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(grid), d)
    m_ref = oracle.convolve(oracle_grid(grid), oracle_response(resp), s_ref)
    assert relL2_per_channel(m, m_ref) < TOL_FRAME


def test_dense_event_routing(pctx):
    """configs[4]-style dense event (1M depos on the MicroBooNE U plane): AUTO
    keeps the time-domain kernel (2.3x faster than the row FFT at this
    density, round 2), a smaller kappa sends it to the row FFT, and the two
    kernels agree within the tolerance."""
    grids, resps = microboone_grids()
    d = microboone_event(1_000_000, seed=3)[0]
    plane = Plane(pctx, grids[0], resps[0])
    res = plane.simulate(d, SimConfig(fluctuate=False))
    assert res.timing["direct_planes"] == 1  # AUTO -> time domain
    pctx.set_direct_kappa(16.0)
    try:
        res_fft = plane.simulate(d, SimConfig(fluctuate=False))
    finally:
        pctx.set_direct_kappa(128.0)
    assert res_fft.timing["direct_planes"] == 0  # the work estimate past 16 x cells -> row FFT
    assert relL2_per_channel(res.frame, res_fft.frame) < TOL_FRAME
    # and the 100k-depo event stays on the time-domain kernel
    res2 = plane.simulate(microboone_event(100_000, seed=1)[0], SimConfig(fluctuate=False))
    assert res2.timing["direct_planes"] == 1


@pytest.mark.parametrize("kind", ["collection", "induction"])
def test_direct_wide_and_narrow_depos(pctx, oracle, kind):
    """Tick profiles wider than 32 bins (sigma_t 3-6 us: the scalar path of the
    response-profile kernel, profiles longer than a warp's 160 register taps:
    k_direct's general path) and depos narrower than a quarter bin (the fp64
    fallback of the fp32 sampler), mixed with ordinary ones, on the forced
    time-domain path."""
    resp = ResponseParams(plane_kind=kind, wire_weights=(0.1, 1.0, 0.1) if kind == "induction" else (1.0,))
    depos = line_tracks(600, SMALL, seed=8)
    depos["sigma_t"][::7] = np.linspace(3.0, 6.0, len(depos[::7]))
    depos["sigma_x"][3::11] = 0.2   # < pitch / 4
    depos["sigma_t"][5::13] = 0.05  # < tick / 4
    m = _frame(pctx, "direct", SMALL, resp, depos)
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(SMALL), depos)
    m_ref = oracle.convolve(oracle_grid(SMALL), oracle_response(resp), s_ref)
    assert relL2_per_channel(m, m_ref) < TOL_FRAME
    m_fft = _frame(pctx, "fft", SMALL, resp, depos)
    assert relL2_per_channel(m_fft, m_ref) < TOL_FRAME


@pytest.mark.parametrize("path", ["direct", "fft"])
def test_extreme_charge_range(pctx, oracle, path):
    """Charges from 1 to 1e12 electrons on one plane: segment bounds beyond
    32 bits (k_direct's bound pass re-runs with a coarser unit), per-row
    fixed-point scales spanning ~40 binary orders, and single terms near
    the row's 2^29 budget (k_direct rounds each term with one DFMA, exact
    for |term| < 2^51)."""
    resp = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))
    depos = line_tracks(600, SMALL, seed=12)
    rng = np.random.default_rng(12)
    depos["q"] = np.round(10.0 ** rng.uniform(0.0, 12.0, len(depos))).astype(np.int64)
    depos["q"][::50] = 10**12
    m = _frame(pctx, path, SMALL, resp, depos)
    s_ref, _ = oracle.charge_fluct_off(oracle_grid(SMALL), depos)
    m_ref = oracle.convolve(oracle_grid(SMALL), oracle_response(resp), s_ref)
    assert np.isfinite(m).all()
    assert relL2_per_channel(m, m_ref) < TOL_FRAME


def test_untimed_device_event_equals_timed(pctx):
    """The untimed device path chains its three kernels with programmatic
    dependent launches (the profile and tile kernels start while their
    predecessor drains); its frames must equal the timed host path's bitwise,
    call after call."""
    import torch
    from paper_2104_08265_b200 import simulate_event_device
    grids, resps = microboone_grids()
    planes = [Plane(pctx, g, r) for g, r in zip(grids, resps)]
    ev = microboone_event(100_000, seed=21)
    cfg = SimConfig(fluctuate=False)
    want = [p.simulate(d, SimConfig(grid=g, response=r, fluctuate=False)).frame
            for p, d, g, r in zip(planes, ev, grids, resps)]
    dev = [torch.from_numpy(d.view(np.uint8)).cuda() for d in ev]
    frames = [torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes]
    for _ in range(3):
        simulate_event_device(pctx, planes, dev, [len(d) for d in ev], cfg, frames)
        pctx.synchronize()
        for f, w in zip(frames, want):
            assert np.array_equal(f.cpu().numpy(), w)
    # back to back without synchronisation (each call's sampler launched
    # programmatically behind the previous call's k_direct): A, B, A
    ev_b = microboone_event(60_000, seed=22)
    want_b = [p.simulate(d, SimConfig(grid=g, response=r, fluctuate=False)).frame
              for p, d, g, r in zip(planes, ev_b, grids, resps)]
    dev_b = [torch.from_numpy(d.view(np.uint8)).cuda() for d in ev_b]
    outs = [[torch.empty(p.shape, dtype=torch.float32, device="cuda") for p in planes] for _ in range(3)]
    for k, (dv, e) in enumerate([(dev, ev), (dev_b, ev_b), (dev, ev)]):
        simulate_event_device(pctx, planes, dv, [len(d) for d in e], cfg, outs[k])
    pctx.synchronize()
    for k, w_all in enumerate([want, want_b, want]):
        for f, w in zip(outs[k], w_all):
            assert np.array_equal(f.cpu().numpy(), w)
