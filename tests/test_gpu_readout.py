"""run_simulation's readout on the GPU: add_noise + digitize fused into the
convolution kernels' frame stores (ws_run_simulation / ws_run_events), its
output types (int32 / uint16 ADC, fp32 / fp64 frame), the unfused noise
modes, and the drop-in typed with the reference's own wiresim:: types against
the unmodified reference (SimResult::adc, pipeline.cpp:345-427).

The fused readout must give the same bits as the separate kernels
(ws_noise_digitize_device), which are themselves checked against the oracle
and the reference in test_gpu_noise.py."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2104_08265_b200 import (AdcConfig, Context, GridSpec, NoiseModel, Plane, ResponseParams, RngConfig,
                                   SimConfig, WsError, run_events)
from paper_2104_08265_b200.workloads import line_tracks

from .helpers import oracle_grid, oracle_response, relL2_per_channel

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

GRIDS = {
    "n4": GridSpec(n_wires=96, n_ticks=900, pad_wires=20, pad_ticks=100),    # 1100 ticks: vector stores
    "odd": GridSpec(n_wires=60, n_ticks=601, pad_wires=10, pad_ticks=100),   # 801 ticks: pair stores
}
RESP = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))


def _cfg(grid, noise=None, seed=77, adc=AdcConfig(0.5, 2048.0, 12)):
    return SimConfig(grid=grid, response=RESP, fluctuate=False, rng=RngConfig(seed=seed),
                     noise=noise or NoiseModel(), adc=adc)


def _unfused(ctx, plane, depos, cfg, rng, sigma):
    import torch
    m = plane.simulate(depos, cfg).frame
    fd = torch.from_numpy(m.copy()).cuda()
    adc = torch.empty(m.shape, dtype=torch.int32, device="cuda")
    plane.noise_digitize_device(fd, sigma=sigma, seed=cfg.rng.seed, rng=rng, adc_dev=adc, scale=cfg.adc.scale,
                                offset=cfg.adc.offset, bits=cfg.adc.bits)
    ctx.synchronize()
    return fd.cpu().numpy(), adc.cpu().numpy()


@pytest.mark.parametrize("path", ["direct", "fft"])
@pytest.mark.parametrize("gname", ["n4", "odd"])
@pytest.mark.parametrize("sigma", [0.0, 3.0])
def test_fused_readout_equals_separate_kernels(ctx, path, gname, sigma):
    grid = GRIDS[gname]
    plane = Plane(ctx, grid, RESP)
    depos = line_tracks(400, grid, seed=2)
    cfg = _cfg(grid, NoiseModel(mode="white", sigma=sigma, rng="philox") if sigma else None)
    ctx.set_conv_path(path)
    try:
        frame_ref, adc_ref = _unfused(ctx, plane, depos, cfg, "philox", sigma)
        r = plane.run(depos, cfg, want_frame=True)
    finally:
        ctx.set_conv_path("auto")
    # the same fp64 arithmetic on the same fp32 samples; libm may differ by an
    # ulp between translation units, which moves a code only at an exact tie
    diff = np.abs(r.adc.astype(np.int64) - adc_ref)
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-5
    assert np.max(np.abs(r.frame - frame_ref)) <= 1e-6 * (np.abs(frame_ref).max() + 1.0)
    if sigma == 0.0:
        np.testing.assert_array_equal(r.adc, adc_ref)


def test_output_types(ctx):
    grid = GRIDS["n4"]
    plane = Plane(ctx, grid, RESP)
    depos = line_tracks(400, grid, seed=3)
    cfg = _cfg(grid, NoiseModel(mode="white", sigma=2.0, rng="philox"))
    a = plane.run(depos, cfg, adc_type="i32", want_frame=True, frame_type="f32")
    b = plane.run(depos, cfg, adc_type="u16", want_frame=True, frame_type="f64")
    assert b.adc.dtype == np.uint16 and b.frame.dtype == np.float64
    np.testing.assert_array_equal(a.adc, b.adc.astype(np.int32))
    np.testing.assert_array_equal(a.frame, b.frame.astype(np.float32))  # fp64 = the unrounded noisy sample
    # no noise: the fp64 frame is the fp32 result widened
    c = plane.run(depos, _cfg(grid), want_frame=True, frame_type="f64")
    d = plane.simulate(depos, _cfg(grid)).frame
    np.testing.assert_array_equal(c.frame, d.astype(np.float64))


@pytest.mark.parametrize("mode", ["white", "spectrum"])
def test_unfused_noise_modes(ctx, mode):
    """Substream white noise (sequential per wire) and spectrum noise run as
    a second kernel over the fp32 frame: the same as the separate entry point."""
    import torch
    grid = GridSpec(n_wires=60, n_ticks=600, pad_wires=10, pad_ticks=100)  # 800 ticks: 7-smooth
    plane = Plane(ctx, grid, RESP)
    depos = line_tracks(300, grid, seed=4)
    n = grid.padded_ticks()
    amp = 3.0 / (1.0 + np.minimum(np.arange(n), n - np.arange(n)) / 40.0)
    noise = NoiseModel(mode="white", sigma=2.5) if mode == "white" else NoiseModel(mode="spectrum",
                                                                                      amplitude_spectrum=amp)
    cfg = _cfg(grid, noise, seed=31)
    r = plane.run(depos, cfg, want_frame=True)
    m = plane.simulate(depos, cfg).frame
    fd = torch.from_numpy(m.copy()).cuda()
    adc = torch.empty(m.shape, dtype=torch.int32, device="cuda")
    plane.noise_digitize_device(fd, sigma=2.5 if mode == "white" else 0.0, seed=31, rng="substream", adc_dev=adc,
                                scale=0.5, offset=2048.0, bits=12, spectrum=amp if mode == "spectrum" else None)
    ctx.synchronize()
    np.testing.assert_array_equal(r.frame, fd.cpu().numpy())
    np.testing.assert_array_equal(r.adc, adc.cpu().numpy())


def test_readout_vs_oracle(ctx, oracle):
    """ADC of the full chain against the oracle's (fp64 frame + the same
    substream white noise + digitize): codes move by one only where the fp32
    frame sits next to a rounding boundary."""
    grid = GRIDS["n4"]
    plane = Plane(ctx, grid, RESP)
    depos = line_tracks(500, grid, seed=6)
    cfg = _cfg(grid, NoiseModel(mode="white", sigma=1.5), seed=11, adc=AdcConfig(1.0, 1000.0, 12))
    r = plane.run(depos, cfg, want_frame=True)
    og = oracle_grid(grid)
    s_ref, _ = oracle.charge_fluct_off(og, depos)
    m_ref = oracle.convolve(og, oracle_response(RESP), s_ref)
    noisy = oracle.add_white_noise(og, m_ref, 1.5, 11, rng_mode=0)
    adc_ref = oracle.digitize(noisy, 1.0, 1000.0, 12)
    assert relL2_per_channel(r.frame, noisy) < 1e-5
    diff = np.abs(r.adc.astype(np.int64) - adc_ref)
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-2


def test_run_events_equal_single_runs(ctx):
    grids = [GRIDS["n4"], GridSpec(n_wires=120, n_ticks=900, pad_wires=20, pad_ticks=100)]
    planes = [Plane(ctx, g, RESP) for g in grids]
    cfg = _cfg(grids[0], NoiseModel(mode="white", sigma=1.0, rng="philox"))
    events = [[line_tracks(300 + 50 * e, g, seed=20 + e + 7 * i) for i, g in enumerate(grids)] for e in range(5)]
    adcs, frames, _ = run_events(ctx, planes, events, cfg, adc_type="u16", want_frame=True)
    for e, ev in enumerate(events):
        for i, (p, d) in enumerate(zip(planes, ev)):
            one = p.run(d, cfg, adc_type="u16", want_frame=True)
            np.testing.assert_array_equal(adcs[e][i], one.adc)
            np.testing.assert_array_equal(frames[e][i], one.frame)


def test_readout_errors(ctx):
    grid = GRIDS["n4"]
    plane = Plane(ctx, grid, RESP)
    depos = line_tracks(50, grid, seed=1)
    with pytest.raises(WsError) as e:
        plane.run(depos, _cfg(grid, adc=AdcConfig(1.0, 0.0, 17)))
    assert e.value.code == 1 and "bits" in str(e.value)
    with pytest.raises(WsError) as e:
        plane.run(depos, _cfg(grid, NoiseModel(mode="white", sigma=-1.0)))
    assert e.value.code == 1 and "sigma" in str(e.value)
    with pytest.raises(WsError) as e:
        plane.run(depos, _cfg(grid, NoiseModel(mode="spectrum", amplitude_spectrum=np.ones(5))))
    assert e.value.code == 1 and "amplitude_spectrum" in str(e.value)


def test_dropin_reference_types():
    """include/wiresim_b200_dropin.hpp with a real wiresim::SimConfig and
    std::vector<wiresim::Depo>, against wiresim::run_simulation in the same
    process (oracle/_ref/dropin_ref, built where the reference exists): the
    integer charge grid and clipped charge identical, ADC within one code at
    rounding boundaries, the reference's exception type for a bad config."""
    exe = ROOT / "oracle" / "_ref" / "dropin_ref"
    if not exe.exists():
        pytest.skip("oracle/_ref/dropin_ref not built (needs /root/reference at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    cases = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(cases) >= 7, r.stdout + r.stderr
    bad = [c for c in cases if not c["ok"]]
    assert r.returncode == 0 and not bad, r.stdout + r.stderr
