"""Pin the CPU oracle (oracle/wsoracle.c) before trusting it.

1. Against the committed golden vectors produced by the UNMODIFIED reference
   (tests/golden/make_golden.py through oracle/_ref) — runs everywhere.
2. Against the live reference library when oracle/_ref/libwsref.so exists.
3. SPEC.md acceptance properties that pin the hot path (AC1, AC4, AC5, AC10).
"""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import DEPO_DTYPE, Drift, make_grid, make_response

GOLD = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())
ARR = np.load(Path(__file__).parent / "golden" / "golden_arrays.npz")


def _fnv(oracle, a):
    a = np.ascontiguousarray(a)
    return int(oracle.lib.wso_fnv1a64(a.ctypes.data, a.nbytes))


def _small_grid():
    g = GOLD["grid_small"]
    return make_grid(g["n_wires"], g["n_ticks"], g["pad_wires"], g["pad_ticks"], g["pitch"], g["tick"])


def _edge_depos():
    e = GOLD["edge_depos"]
    d = np.zeros(len(e["id"]), dtype=DEPO_DTYPE)
    for k in d.dtype.names:
        d[k] = e[k]
    return d


# ------------------------------------------------------------------ golden --
def test_philox_kat(oracle):
    for kat in GOLD["philox_kat"]:
        assert oracle.philox(kat["ctr"], kat["key"]).tolist() == kat["out"]
    # Random123 published KATs
    assert [hex(x) for x in oracle.philox([0, 0, 0, 0], [0, 0])] == ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    assert [hex(x) for x in oracle.philox([0, 0, 0, 0], [12345, 0])] == ["0xd1fa3e81", "0x2f7fea51", "0xd2ca9611",
                                                                        "0xe328bbe0"]


def test_draws_golden(oracle):
    for d in GOLD["draws"]:
        assert oracle.draws(d["mode"], 0, d["seed"], d["id"], 8).tolist() == d["uniform"]
        assert oracle.draws(d["mode"], 1, d["seed"], d["id"], 8).tolist() == d["normal"]


def test_binomial_golden(oracle):
    for b in GOLD["binomial"]:
        assert oracle.binomials(b["n"], b["p"], b["seed"], b["id"], 16).tolist() == b["k"]


def test_footprint_and_patch_golden(oracle):
    g = _small_grid()
    d = _edge_depos()
    for i in range(len(d)):
        assert oracle.map_depo(g, d[i]).tolist() == GOLD["map_depo"][i]
        p = oracle.sample_patch(g, d[i])
        gp = GOLD["sample_patch"][i]
        for k in ("wire_offset", "tick_offset", "n_w", "n_t", "clipped"):
            assert p[k] == gp[k], (i, k)
        assert p["values"].ravel().tolist() == gp["values"]  # bit-exact doubles
        assert p["captured_mass"] == gp["captured_mass"]
    assert oracle.map_depo(make_grid(100, 100, 0, 0, 5.0, 1.0),
                           np.array([(0, 10.2, 25.6, 0, 3.3, 1.0)], dtype=DEPO_DTYPE)).tolist() == GOLD["map_depo_spec"]
    # sigma_t 3.3 us, tick 1 us, n_sigma 3 -> 21 ticks
    lo, hi = GOLD["map_depo_spec"][4], GOLD["map_depo_spec"][5]
    assert hi - lo + 1 == 21


def test_drift_golden(oracle):
    d = np.zeros(1, dtype=DEPO_DTYPE)
    d["x"], d["t"] = 100.0, 5.0
    out = oracle.drift(d, Drift(0.0, 1.6, 0.0068, 0.0088))
    for k, v in GOLD["drift_spec"].items():
        assert out[k][0] == v
    assert abs(out["sigma_x"][0] - 1.0488) < 1e-4


def test_small_run_golden(oracle):
    g = _small_grid()
    depos = ARR["small_depos"].view(DEPO_DTYPE)
    s, clipped = oracle.charge_fluct_on(g, depos, rng_mode=0, seed=12345)
    assert np.array_equal(s, ARR["small_charge_substream"])
    assert clipped == GOLD["small_clipped_substream"]
    s, _ = oracle.charge_fluct_on(g, depos, rng_mode=1, seed=12345)
    assert np.array_equal(s, ARR["small_charge_philox"])
    off, clipped = oracle.charge_fluct_off(g, depos)
    assert np.array_equal(off, ARR["small_charge_off"])
    assert clipped == GOLD["small_clipped_off"]
    for name, r in [("collection", make_response()), ("induction", make_response("induction")),
                    ("ww3", make_response("collection", wire_weights=(0.25, 1.0, 0.25)))]:
        m = oracle.convolve(g, r, off)
        ref = ARR[f"small_m_off_{name}"]
        assert np.abs(m - ref).max() <= 1e-12 * np.abs(ref).max()
        m = oracle.convolve(g, r, ARR["small_charge_substream"].astype(np.float64))
        ref = ARR[f"small_m_on_{name}"]
        assert np.abs(m - ref).max() <= 1e-12 * np.abs(ref).max()
        td = oracle.response_td(g, r)
        assert [td["support_ticks"], td["support_wires"]] == GOLD[f"support_{name}"]
    # white noise + digitize (spectral.cpp:188-196, :228-238)
    noisy = oracle.add_white_noise(g, ARR["small_m_off_collection"], 2.0, 12345)
    assert np.abs(noisy - ARR["small_noisy_white"]).max() <= 1e-12
    adc = oracle.digitize(ARR["small_noisy_white"])
    assert np.array_equal(adc, ARR["small_adc_white"])


def test_c1_anchor(oracle):
    """SURVEY.md §4 anchor: gen_depos(10000, seed 7) on 480 x 6000, substream seed 12345."""
    from paper_2104_08265_b200.api import GridSpec, gen_depos
    gc1 = make_grid(480, 6000)
    depos = gen_depos(10_000, 7, GridSpec(n_wires=480, n_ticks=6000))  # product's host generator
    assert _fnv(oracle, depos) == GOLD["c1"]["depos_fnv1a"]
    s, clipped = oracle.charge_fluct_on(gc1, depos, rng_mode=0, seed=12345)
    assert _fnv(oracle, s) == GOLD["c1"]["charge_substream_fnv1a"]
    assert int(s.sum()) == GOLD["c1"]["charge_substream_sum"] == 55_135_105
    assert clipped == GOLD["c1"]["clipped"]
    s, _ = oracle.charge_fluct_on(gc1, depos, rng_mode=1, seed=12345)
    assert _fnv(oracle, s) == GOLD["c1"]["charge_philox_fnv1a"]


# ------------------------------------------------------- live reference --
@pytest.mark.ref
def test_live_reference_random(oracle, ref):
    rng = np.random.default_rng(42)
    g = make_grid(64, 400, 16, 100, 4.0, 0.5, origin_x=-3.0, origin_t=1.25)
    d = np.zeros(400, dtype=DEPO_DTYPE)
    d["id"] = np.arange(400) * 977
    d["t"] = rng.uniform(-60, 260, 400)
    d["x"] = rng.uniform(-80, 330, 400)
    d["q"] = rng.integers(0, 20000, 400)
    d["sigma_t"] = rng.choice([0.0, 0.3, 1.0, 2.5], 400)
    d["sigma_x"] = rng.choice([0.0, 1.0, 4.0, 9.0], 400)
    for i in range(0, 400, 7):
        a, b = oracle.sample_patch(g, d[i]), ref.sample_patch(g, d[i])
        assert a["values"].tobytes() == b["values"].tobytes() and a["wire_offset"] == b["wire_offset"]
    for mode in (0, 1):
        so, co = oracle.charge_fluct_on(g, d, rng_mode=mode, seed=99)
        if mode == 0:
            r = ref.run_simulation(g, make_response(), d, seed=99)
            sr, cr = r["charge"], r["clipped_charge"]
        else:
            sr, cr = ref.charge_fluct_philox(g, d, seed=99)
        assert np.array_equal(so, sr) and co == cr
    so, _ = oracle.charge_fluct_off(g, d)
    sr, _ = ref.charge_fluct_off(g, d)
    assert np.array_equal(so, sr)
    for n, p in [(20, 0.3), (10000, 0.45), (300000, 0.02), (2000, 0.9999)]:
        assert np.array_equal(oracle.binomials(n, p, 5, 11, 64), ref.binomials(n, p, 5, 11, 64))


@pytest.mark.ref
def test_live_reference_drift_and_convolve(oracle, ref):
    g = make_grid(40, 300, 10, 100, 5.0, 0.5)
    d = ref.gen_depos(300, 3, g)
    dp = Drift(-10.0, 1.6, 0.0068, 0.0088)
    assert oracle.drift(d, dp).tobytes() == ref.drift(d, dp).tobytes()
    so, _ = oracle.charge_fluct_off(g, d, drift=dp)
    sr, _ = ref.charge_fluct_off(g, d, drift=dp)
    assert np.array_equal(so, sr)
    for r in (make_response("induction", shaper_order=3, wire_weights=(0.1, -0.2, 1.0, -0.2, 0.1)),
              make_response("collection", field_sigma_t=0.0, shaper_peaking=0.0, gain=3.0)):
        m_o = oracle.convolve(g, r, so)
        m_r = ref.convolve_real(g, r, so)
        assert np.abs(m_o - m_r).max() <= 1e-12 * np.abs(m_r).max()


# ------------------------------------------------------ SPEC properties --
def test_spec_ac4_bruteforce_convolution(oracle):
    """AC4: FFT/circular convolution vs a direct double sum on 16x16."""
    g = make_grid(8, 8, 4, 4, 5.0, 2.0)
    r = make_response("induction", field_sigma_t=1.0, shaper_peaking=0.0, wire_weights=(0.2, 1.0, -0.3))
    td = oracle.response_td(g, r)
    rng = np.random.default_rng(0)
    for _ in range(10):
        s = rng.normal(size=(16, 16))
        m = oracle.convolve(g, r, s)
        ww = np.array([0.2, 1.0, -0.3])
        k = np.zeros((16, 16))
        for dw in (-1, 0, 1):
            for i, c in enumerate(td["kernel"]):
                k[dw % 16, (td["lo_lag"] + i) % 16] += ww[dw + 1] * c
        direct = np.zeros((16, 16))
        for a in range(16):
            for b in range(16):
                direct += k[a, b] * np.roll(np.roll(s, a, 0), b, 1)
        assert np.abs(m - direct).max() <= 1e-10 * np.abs(direct).max()


def test_spec_ac10_response_shapes(oracle):
    g = make_grid(10, 300, 2, 100, 5.0, 0.5)
    ind = oracle.response_td(g, make_response("induction"))
    col = oracle.response_td(g, make_response("collection"))
    assert abs(ind["kernel"].sum()) <= 1e-9 * np.abs(ind["kernel"]).max()
    assert abs(col["kernel"].sum() - 14.0) <= 1e-9


def test_spec_ac1_ac5_conservation_and_mass(oracle):
    from scipy import integrate
    from scipy.special import erf
    g = _small_grid()
    d = ARR["small_depos"].view(DEPO_DTYPE)
    s, clipped = oracle.charge_fluct_on(g, d, rng_mode=0, seed=12345)
    assert int(s.sum()) == int(d["q"].sum()) - clipped  # AC1: exact integers
    rng = np.random.default_rng(5)
    for i in rng.choice(len(d), 20, replace=False):  # AC5
        p = oracle.sample_patch(g, d[i])
        assert p["captured_mass"] >= 0.995 or p["clipped"]
        # un-renormalised bins vs quadrature of the separable Gaussian
        unnorm = p["values"] * p["captured_mass"]
        wl = (p["wire_offset"] - 12) * 5.0
        tl = (p["tick_offset"] - 100) * 0.5
        for a in range(0, p["n_w"], 3):
            for b in range(0, p["n_t"], 4):
                fx = integrate.quad(lambda x: np.exp(-0.5 * ((x - d["x"][i]) / d["sigma_x"][i]) ** 2), wl + 5 * a,
                                    wl + 5 * (a + 1))[0] / (d["sigma_x"][i] * np.sqrt(2 * np.pi))
                ft = 0.5 * (erf((tl + 0.5 * (b + 1) - d["t"][i]) / (np.sqrt(2) * d["sigma_t"][i])) -
                            erf((tl + 0.5 * b - d["t"][i]) / (np.sqrt(2) * d["sigma_t"][i])))
                assert abs(unnorm[a, b] - fx * ft) <= 1e-9


def test_impact_restatement_pins_to_wire_binning(oracle):
    """oracle.impact_charge (sampling at impact resolution, the checker of
    ws_plane_create_impacts) with one class equals the oracle's wire binning,
    which is pinned to the reference: the telescoping the degenerate case
    relies on."""
    from oracle.oracle import impact_charge
    from paper_2104_08265_b200 import GridSpec
    from paper_2104_08265_b200.workloads import line_tracks
    from .helpers import oracle_grid
    grid = GridSpec(n_wires=96, n_ticks=900, pad_wires=20, pad_ticks=100, pitch=5.0, tick=0.5)
    d = line_tracks(300, grid, seed=5)
    d["sigma_x"][:10] = 0.0  # delta depos: the containing sub-bin
    (s,), clipped = impact_charge(oracle_grid(grid), d, 10, [(1 << 10) - 1])
    s_ref, clipped_ref = oracle.charge_fluct_off(oracle_grid(grid), d)
    assert clipped == clipped_ref
    np.testing.assert_allclose(s, s_ref, rtol=0, atol=1e-9 * s_ref.max())
