"""The tensor-core convolution of a given charge grid (k_conv_tc,
ws_conv_tc.cu) against the oracle's direct circular convolution (convolve,
spectral.cpp:141-175): float grids through ws_convolve_device over stencil
widths (1, 3, 5 taps; 7 taps runs the row FFT), tick counts that are odd or
not a multiple of the 128-tick sub-block, grids narrower than one tile in
both directions, delta responses (a one-tap kernel), and values far beyond
the 11-bit TF32 integer range (the hi/lo split of a float grid)."""
import numpy as np
import pytest

from paper_2104_08265_b200 import GridSpec, Plane, ResponseParams

from .helpers import oracle_grid, oracle_response, relL2_per_channel

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["tc2", "tc2_cpasync", "tc1"], autouse=True)
def tc_kernel(request, monkeypatch):
    """Every case through the pipelined kernel (k_conv_tc2: TMA slab loads where
    the plane allows them, else cp.async), its cp.async loader forced
    (WS_CONV_TC2_TMA=0), and the one-tile-at-a-time kernel (k_conv_tc,
    WS_CONV_TC2=0)."""
    if request.param == "tc1":
        monkeypatch.setenv("WS_CONV_TC2", "0")
    if request.param == "tc2_cpasync":
        monkeypatch.setenv("WS_CONV_TC2_TMA", "0")
    return request.param


def _conv(ctx, oracle, grid, resp, s):
    import torch
    plane = Plane(ctx, grid, resp)
    sd = torch.from_numpy(np.ascontiguousarray(s, dtype=np.float32)).cuda()
    md = torch.full_like(sd, float("nan"))
    torch.cuda.synchronize()
    plane.convolve_device(sd, md)
    ctx.synchronize()
    m = md.cpu().numpy()
    m_ref = oracle.convolve(oracle_grid(grid), oracle_response(resp), s.astype(np.float32).astype(np.float64))
    assert np.isfinite(m).all()
    return relL2_per_channel(m, m_ref)


@pytest.mark.parametrize("ww", [(1.0,), (0.15, 1.0, 0.15), (-0.05, 0.2, 1.0, 0.2, -0.05),
                                (0.01, -0.05, 0.2, 1.0, 0.2, -0.05, 0.01)])
@pytest.mark.parametrize("kind", ["collection", "induction"])
def test_grid_convolution_stencils(ctx, oracle, ww, kind):
    grid = GridSpec(n_wires=150, n_ticks=1000, pad_wires=20, pad_ticks=100)
    rng = np.random.default_rng(len(ww))
    s = np.zeros((grid.padded_wires(), grid.padded_ticks()))
    s[5:170, :] = rng.integers(0, 300, size=(165, grid.padded_ticks())) * (rng.random((165, grid.padded_ticks())) < 0.3)
    s[0, :50] = 7.0    # wraps in wires and ticks
    s[-1, -40:] = 11.0
    assert _conv(ctx, oracle, grid, ResponseParams(plane_kind=kind, wire_weights=ww), s) < 1e-5


@pytest.mark.parametrize("n_wires,n_ticks,pad", [(7, 301, 3), (40, 97, 5), (33, 1, 0), (300, 2049, 100)])
def test_grid_convolution_shapes(ctx, oracle, n_wires, n_ticks, pad):
    grid = GridSpec(n_wires=n_wires, n_ticks=n_ticks, pad_wires=pad, pad_ticks=pad)
    rng = np.random.default_rng(n_ticks)
    s = rng.integers(0, 100, size=(grid.padded_wires(), grid.padded_ticks())).astype(np.float64)
    resp = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))
    try:
        r = _conv(ctx, oracle, grid, resp, s)
    except Exception as e:  # the reference's own rule: the kernel must fit the padded ticks
        assert "kernel" in str(e) or "support" in str(e), e
        return
    assert r < 1e-5


def test_grid_convolution_delta_response_and_large_values(ctx, oracle):
    grid = GridSpec(n_wires=64, n_ticks=700, pad_wires=10, pad_ticks=120)
    rng = np.random.default_rng(5)
    s = rng.random((grid.padded_wires(), grid.padded_ticks())) * 3e7  # far past 2^11: hi + lo parts
    for fs, sp in [(0.0, 0.0), (0.0, 2.0), (1.0, 0.0)]:
        resp = ResponseParams(plane_kind="collection", field_sigma_t=fs, shaper_peaking=sp)
        assert _conv(ctx, oracle, grid, resp, s) < 1e-5


@pytest.mark.parametrize("q_hot", [60_000_000, 150_000_000])
def test_fluctuation_counts_past_2_11_and_2_22(ctx, oracle, q_hot):
    """Fluctuation-on frames (the walk's integer counts into the grid
    convolution) with cells far past 2^11 and 2^22 electrons: counts below
    2^22 enter exactly as two TF32 halves, larger ones within 2^-22. With
    1.5e8-electron depos the plane carries more than 2^32 electrons, so the
    count grid takes u64 cells (u32 otherwise): both widths, every loader."""
    from paper_2104_08265_b200 import RngConfig, SimConfig
    from paper_2104_08265_b200.workloads import line_tracks
    grid = GridSpec(n_wires=180, n_ticks=900, pad_wires=20, pad_ticks=100, pitch=5.0, tick=0.5)
    d = line_tracks(600, grid, seed=3)
    d["q"][:40] = q_hot  # narrow, hot depos: cells of ~1e7 (or ~3e8) electrons
    d["sigma_t"][:40] = 0.3
    d["sigma_x"][:40] = 2.0
    d["q"][40:200] = 200_000
    resp = ResponseParams(plane_kind="induction", wire_weights=(1.0,), shaper_peaking=2.0)
    cfg = SimConfig(grid=grid, response=resp, fluctuate=True, rng=RngConfig(mode="philox", seed=8))
    res = Plane(ctx, grid, resp).simulate(d, cfg, want_charge=True)
    # (the draws of these depos take binomial's normal branch, where libm ulps
    # may move a count by a few electrons: test_gpu_overflow pins those; here
    # the convolution of the grid the walk produced is checked)
    s = res.charge.astype(np.int64)
    assert s.max() > 2 ** 22 and ((s > 2 ** 11) & (s < 2 ** 22)).any()
    m_ref = oracle.convolve(oracle_grid(grid), oracle_response(resp), s.astype(np.float64))
    assert relL2_per_channel(res.frame, m_ref) < 1e-5
