"""BASELINE.json configs beyond the headline event, as parity / property tests
(SURVEY.md §8(d)-(e)):

* configs[3] (C4): a ProtoDUNE-SP-style event, 12 anode faces x U/V/W
  (800/800/480 channels x 6000 ticks) as 36 independent planes, sharded over
  "ranks" (separate contexts standing in for GPUs) by the LPT cost model. The
  union of the shards equals the single-context run bit for bit
  (placement invariance), and sampled planes match the oracle.
* configs[4] (C5): batched events through the pipelined host path
  (ws_simulate_events), 64 events, each frame bitwise equal to its own
  single-event call; the 1k-1M depos/event sweep on the MicroBooNE geometry
  conserves charge and is run-to-run deterministic.
* configs[2] (C3): fluctuation on with the shared Philox stream and the
  electronics response on the MicroBooNE U plane (exact integer charge vs the
  oracle at reduced depo count; the full-size timing is tools/fluct_time.py).
"""
import numpy as np
import pytest

from paper_2104_08265_b200 import Context, GridSpec, Plane, ResponseParams, RngConfig, SimConfig, simulate_event, \
    simulate_events
from paper_2104_08265_b200.sharding import protodune_units, shard_units, unit_cost
from paper_2104_08265_b200.workloads import line_tracks, microboone_event, microboone_grids

from .helpers import oracle_grid, oracle_response, relL2_per_channel

pytestmark = pytest.mark.gpu

TOL_FRAME = 1e-5


def _pd_grid(wires):
    return GridSpec(n_wires=wires, n_ticks=6000, pad_wires=100, pad_ticks=100, pitch=5.0, tick=0.5)


def _pd_event(n_per_plane=2000):
    units = protodune_units()
    kinds = ("induction", "induction", "collection")
    wires = (800, 800, 480)
    grids = [_pd_grid(wires[p]) for _, p, _, _ in units]
    resps = [ResponseParams(plane_kind=kinds[p], wire_weights=(0.1, 1.0, 0.1) if p < 2 else (1.0,))
             for _, p, _, _ in units]
    depos = [line_tracks(n_per_plane, g, seed=100 + i) for i, g in enumerate(grids)]
    return units, grids, resps, depos


def _run_units(ctx, idx, grids, resps, depos, cfg):
    """Units idx through one context, grouped 3 planes per launch (one face)."""
    planes = [Plane(ctx, grids[i], resps[i]) for i in idx]
    out = {}
    for k in range(0, len(idx), 3):
        chunk = list(range(k, min(k + 3, len(idx))))
        frames, _ = simulate_event(ctx, [planes[j] for j in chunk], [depos[idx[j]] for j in chunk], cfg)
        for j, f in zip(chunk, frames):
            out[idx[j]] = f
    for p in planes:
        p.close()
    return out


def test_protodune_faces_sharded_placement_invariant(oracle):
    units, grids, resps, depos = _pd_event()
    cfg = SimConfig(fluctuate=False)
    ctx = Context(0)
    whole = _run_units(ctx, list(range(len(units))), grids, resps, depos, cfg)
    ctx.close()
    costs = [unit_cost(w, t, len(depos[i])) for i, (_, _, w, t) in enumerate(units)]
    for world in (2, 4, 8):
        merged = {}
        for owned in shard_units(costs, world):
            c = Context(0)  # one "rank"
            merged.update(_run_units(c, owned, grids, resps, depos, cfg))
            c.close()
        assert sorted(merged) == list(range(len(units)))
        for i in range(len(units)):
            assert np.array_equal(merged[i], whole[i]), f"unit {units[i][:2]} differs at world {world}"
    # two sampled planes (an induction U and a collection W) against the oracle
    for i in (0, 5):
        og = oracle_grid(grids[i])
        s, _ = oracle.charge_fluct_off(og, depos[i])
        m_ref = oracle.convolve(og, oracle_response(resps[i]), s)
        assert relL2_per_channel(whole[i], m_ref) < TOL_FRAME


def test_batched_events_equal_single_calls():
    grid = GridSpec(n_wires=200, n_ticks=2000, pad_wires=20, pad_ticks=100)
    resp = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))
    cfg = SimConfig(fluctuate=False)
    ctx = Context(0)
    plane = Plane(ctx, grid, resp)
    events = [[line_tracks(1000, grid, seed=7 + e)] for e in range(64)]
    frames, _ = simulate_events(ctx, [plane], events, cfg)
    for e in (0, 1, 31, 63):
        single = plane.simulate(events[e][0], cfg).frame
        assert np.array_equal(frames[e][0], single)
    plane.close()
    ctx.close()


@pytest.mark.parametrize("n_depos", [1_000, 10_000, 100_000, 1_000_000])
def test_microboone_sweep_charge_and_determinism(n_depos):
    """configs[4]'s per-event sizes on the MicroBooNE geometry: the charge grid
    sums to sum(q) - clipped (1e-6), and two runs give identical frames."""
    grids, resps = microboone_grids()
    ctx = Context(0)
    plane = Plane(ctx, grids[2], resps[2])  # W, 3456 wires
    d = microboone_event(n_depos, seed=11)[2]
    cfg = SimConfig(grid=grids[2], response=resps[2], fluctuate=False)
    a = plane.simulate(d, cfg, want_charge=True)
    want = float(d["q"].sum()) - a.timing["clipped_charge"]
    assert abs(float(a.charge.sum(dtype=np.float64)) - want) <= 1e-6 * want
    b = plane.simulate(d, cfg)
    c = plane.simulate(d, cfg)
    assert np.array_equal(b.frame, c.frame)
    plane.close()
    ctx.close()


def test_fluct_on_philox_with_shaper_microboone_u(oracle):
    """configs[2]: Philox fluctuation + electronics response (shaper on) on the
    MicroBooNE U plane geometry; integer charge identical to the oracle."""
    grids, resps = microboone_grids()
    g, r = grids[0], resps[0]
    ctx = Context(0)
    plane = Plane(ctx, g, r)
    d = microboone_event(5000, seed=4)[0]
    cfg = SimConfig(grid=g, response=r, fluctuate=True, rng=RngConfig(mode="philox", seed=12345))
    res = plane.simulate(d, cfg, want_charge=True)
    s_ref, clipped = oracle.charge_fluct_on(oracle_grid(g), d, rng_mode=1, seed=12345)
    assert np.array_equal(res.charge.astype(np.int64), s_ref)
    assert res.timing["clipped_charge"] == clipped
    m_ref = oracle.convolve(oracle_grid(g), oracle_response(r), s_ref.astype(np.float64))
    assert relL2_per_channel(res.frame, m_ref) < TOL_FRAME
    plane.close()
    ctx.close()


def test_multi_device_abi_events_and_units():
    """ws_multi_* (one host thread per context; here two contexts on the one
    GPU of the box): events and (face, plane) units sharded by LPT, outputs
    gathered into the caller's buffers, bitwise equal to one context."""
    from paper_2104_08265_b200 import Multi
    grids, resps, _ = microboone_like_small()
    specs = list(zip(grids, resps))
    cfg = SimConfig(fluctuate=False)
    events = [[line_tracks(500 + 300 * (e % 3), g, seed=40 + 3 * e + i) for i, g in enumerate(grids)]
              for e in range(7)]
    m = Multi([0, 0], specs)
    outs, where = m.run_events(events, cfg)
    assert sorted(set(where)) == [0, 1]
    ctx = Context(0)
    planes = [Plane(ctx, g, r) for g, r in specs]
    for e, ev in enumerate(events):
        for i, d in enumerate(ev):
            np.testing.assert_array_equal(outs[e][i], planes[i].simulate(d, cfg).frame)
    adcs, _ = m.run_events(events[:3], cfg, adc_type="u16")
    for e in range(3):
        for i, d in enumerate(events[e]):
            np.testing.assert_array_equal(adcs[e][i], planes[i].run(d, cfg, adc_type="u16").adc)
    plane_of = [u % len(specs) for u in range(9)]
    depos = [line_tracks(200 + 100 * u, grids[p], seed=90 + u) for u, p in enumerate(plane_of)]
    frames, udev = m.run_units(plane_of, depos, cfg)
    assert sorted(set(udev)) == [0, 1]
    for u, p in enumerate(plane_of):
        np.testing.assert_array_equal(frames[u], planes[p].simulate(depos[u], cfg).frame)
    m.close()
    ctx.close()


def microboone_like_small():
    grids = [GridSpec(n_wires=240, n_ticks=1600, pad_wires=20, pad_ticks=100, pitch=3.0),
             GridSpec(n_wires=240, n_ticks=1600, pad_wires=20, pad_ticks=100, pitch=3.0),
             GridSpec(n_wires=300, n_ticks=1600, pad_wires=20, pad_ticks=100, pitch=3.0)]
    resps = [ResponseParams(plane_kind="induction"), ResponseParams(plane_kind="induction"), ResponseParams()]
    return grids, resps, None
