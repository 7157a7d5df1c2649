"""Impact positions (ws_plane_create_impacts; north star (3), BASELINE.json
configs[0] "10 impacts/pitch").

The reference bins the transverse axis once per wire pitch and stands in for
per-impact responses with one response per plane (core.cpp:31-32,
spectral.cpp:124-135), so it pins only the degenerate case:
identical per-impact responses, whose sub-bin integrals telescope to the
wire-bin integral (SURVEY.md §8(a) "Equivalences"). That case is checked
against the reference-pinned oracle on configs[0] (C1: 480 wires x 6000
ticks, 10k depos, 10 impacts/pitch), on both convolution kernels and with
fluctuation. Distinct per-impact responses are checked against
oracle.impact_charge (a numpy restatement of the sampling at impact
resolution, itself equal to the oracle's wire binning in the degenerate case)
convolved class by class with the oracle's reference-pinned convolution."""
import numpy as np
import pytest

from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, RngConfig, SimConfig, WsError
from paper_2104_08265_b200.workloads import line_tracks

from .helpers import oracle_grid, oracle_response, relL2_per_channel

pytestmark = pytest.mark.gpu

C1 = GridSpec(n_wires=480, n_ticks=6000, pad_wires=100, pad_ticks=100, pitch=5.0, tick=0.5)
SMALL = GridSpec(n_wires=96, n_ticks=900, pad_wires=20, pad_ticks=100, pitch=5.0, tick=0.5)


@pytest.fixture(scope="module")
def c1_ref(oracle):
    resp = ResponseParams(plane_kind="collection")
    d = line_tracks(10_000, C1, seed=1)
    s, clipped = oracle.charge_fluct_off(oracle_grid(C1), d)
    return resp, d, s, clipped, oracle.convolve(oracle_grid(C1), oracle_response(resp), s)


@pytest.mark.parametrize("path", ["direct", "fft"])
def test_c1_ten_identical_impacts_equal_reference(ctx, c1_ref, path):
    resp, d, s_ref, clipped, m_ref = c1_ref
    p10 = Plane(ctx, C1, resp, impacts_per_pitch=10)
    assert p10.info["impacts_per_pitch"] == 10 and p10.info["n_response_classes"] == 1
    ctx.set_conv_path(path)
    try:
        r = p10.simulate(d, SimConfig(grid=C1, response=resp, fluctuate=False))
    finally:
        ctx.set_conv_path("auto")
    assert relL2_per_channel(r.frame, m_ref) < 1e-5
    assert r.timing["clipped_charge"] == clipped
    one = Plane(ctx, C1, resp).simulate(d, SimConfig(grid=C1, response=resp, fluctuate=False))
    assert relL2_per_channel(r.frame, one.frame) < 1e-5


def test_c1_impacts_charge_and_fluctuation(ctx, c1_ref, oracle):
    resp, d, s_ref, clipped, _ = c1_ref
    p10 = Plane(ctx, C1, resp, impacts_per_pitch=10)
    s = p10.simulate(d, SimConfig(grid=C1, response=resp, fluctuate=False), want_charge=True).charge
    assert relL2_per_channel(s, s_ref) < 1e-5
    q = float(d["q"].sum()) - clipped
    assert abs(float(s.astype(np.float64).sum()) - q) <= 1e-6 * q
    # fluctuation: the wire profile is the fp64 sum of the sub-bin integrals
    # (equal to the wire-bin integral up to rounding): the same walk, with
    # at most rare one-ulp-driven draw differences
    sub = d[:2000]
    cfg = SimConfig(grid=C1, response=resp, fluctuate=True, rng=RngConfig(mode="philox", seed=7))
    got = p10.simulate(sub, cfg, want_charge=True).charge.astype(np.int64)
    want, _ = oracle.charge_fluct_on(oracle_grid(C1), sub, rng_mode=1, seed=7)
    assert got.sum() == want.sum()
    assert np.abs(got - want).sum() <= 1e-4 * want.sum()


def _two_class_responses():
    a = ResponseParams(plane_kind="induction", field_sigma_t=1.0, wire_weights=(0.1, 1.0, 0.1))
    b = ResponseParams(plane_kind="induction", field_sigma_t=1.1, wire_weights=(0.25, 1.0, 0.25))
    return [a, b, b, a], (0b1001, 0b0110), (a, b)  # edges vs centre of the pitch


@pytest.mark.parametrize("n_depos", [600, 4000])
def test_distinct_impact_responses_vs_restatement(ctx, oracle, n_depos):
    resps, masks, classes = _two_class_responses()
    d = line_tracks(n_depos, SMALL, seed=9)
    d["sigma_x"][:20] = 0.0
    d["sigma_x"][20:40] = 0.4  # narrower than a quarter pitch: the fp64 sampler
    plane = Plane(ctx, SMALL, resps, impacts_per_pitch=4)
    assert plane.info["n_response_classes"] == 2
    r = plane.simulate(d, SimConfig(grid=SMALL, fluctuate=False))
    assert r.timing["direct_planes"] == 1
    og = oracle_grid(SMALL)
    from oracle.oracle import impact_charge
    s_c, clipped = impact_charge(og, d, 4, masks)
    m_ref = sum(oracle.convolve(og, oracle_response(rc), s) for rc, s in zip(classes, s_c))
    assert relL2_per_channel(r.frame, m_ref) < 1e-5
    assert r.timing["clipped_charge"] == clipped
    # in an event with other planes, and through the readout path
    other = Plane(ctx, SMALL, ResponseParams())
    from paper_2104_08265_b200 import simulate_event
    frames, _ = simulate_event(ctx, [other, plane, other], [d, d, d], SimConfig(fluctuate=False))
    np.testing.assert_array_equal(frames[1], r.frame)
    ro = plane.run(d, SimConfig(grid=SMALL, fluctuate=False), want_frame=True)
    np.testing.assert_array_equal(ro.frame, r.frame)


def test_impact_errors(ctx):
    resps, _, _ = _two_class_responses()
    with pytest.raises(WsError) as e:
        Plane(ctx, SMALL, ResponseParams(), impacts_per_pitch=33)
    assert e.value.code == 1 and "impacts_per_pitch" in str(e.value)
    plane = Plane(ctx, SMALL, resps, impacts_per_pitch=4)
    d = line_tracks(100, SMALL, seed=1)
    with pytest.raises(WsError) as e:
        plane.simulate(d, SimConfig(fluctuate=True))
    assert e.value.code == 1 and "fluctuation" in str(e.value)
    ctx.set_conv_path("fft")
    try:
        with pytest.raises(WsError) as e:
            plane.simulate(d, SimConfig(fluctuate=False))
        assert e.value.code == 1 and "time-domain" in str(e.value)
    finally:
        ctx.set_conv_path("auto")
