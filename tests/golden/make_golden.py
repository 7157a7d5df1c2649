"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It builds oracle/_ref/libwsref.so (oracle/Makefile `ref`) and records, through
ref_harness.cpp, known-answer vectors for every function on the hot path.
The fixtures are small, committed, and read by tests/test_oracle.py (CPU) and
tests/test_gpu_parity.py (GPU box, where /root/reference does not exist).
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import DEPO_DTYPE, Drift, Reference, build_ref, fnv1a64, make_grid, make_response  # noqa: E402


def edge_depos():
    """Depos exercising the footprint / clip / delta / empty rules."""
    d = np.zeros(12, dtype=DEPO_DTYPE)
    d["id"] = np.arange(12)
    d["t"] = [10.2, 0.0, 149.75, -49.9, 1e5, 75.0, 33.3, 120.0, 0.25, 80.0, 149.99, 60.0]
    d["x"] = [25.6, 0.0, 239.9, -1e4, 120.0, 60.0, 2.5, 100.0, 238.0, -3.0, 119.0, 77.7]
    d["q"] = [5000, 1200, 9999, 3000, 4000, 0, 1, 2500, 7000, 6000, 8000, 100]
    d["sigma_t"] = [1.1, 0.5, 1.5, 1.0, 0.0, 0.7, 3.3, 0.01, 1.2, 0.9, 2.0, 0.6]
    d["sigma_x"] = [3.0, 2.5, 7.5, 5.0, 4.0, 0.0, 6.0, 5.5, 2.6, 4.4, 0.001, 3.3]
    return d


CSV_CASES = {
    "ok_blank_lines": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1.5,2.5,100,0.5,3\n\n1,+2,  3.25,7,1e-1,0\n",
    "no_trailing_newline": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,3,4,5",
    "header_only": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n",
    "empty": "",
    "bad_header": "id,t,x,q,st,sx\n0,1,2,3,4,5\n",
    "crlf": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\r\n0,1,2,3,4,5\r\n",
    "crlf_row": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,3,4,5\r\n",
    "trailing_field": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,3,4,5,6\n",
    "short_row": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,3,4\n",
    "text_field": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,abc,3,4,5\n",
    "float_charge": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,3.5,4,5\n",
    "id_gap": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,3,4,5\n2,1,2,3,4,5\n",
    "negative_charge": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,-3,4,5\n",
    "negative_width": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,1,2,3,4,-5\n",
    "zero_width": "id,t_us,x_mm,q,sigma_t_us,sigma_x_mm\n0,-1e3,-2.5e-7,0,0,0\n",
}


def csv_fixtures(ref):
    """Depo CSV ingestion (load_depos, pipeline.cpp:226-262) and writer
    (gen_depos, pipeline.cpp:264-294): a reference-written file plus the
    reference loader's verdict on edge-case files (path replaced by <path>)."""
    import tempfile
    g = make_grid(48, 300, 12, 100, 5.0, 0.5)
    ref.gen_depos_csv(64, 11, g, HERE / "depos_ref.csv")
    cases = {}
    with tempfile.TemporaryDirectory() as td:
        for name, text in CSV_CASES.items():
            path = Path(td) / f"{name}.csv"
            path.write_bytes(text.encode())
            try:
                d = ref.load_depos(path)
                cases[name] = {"text": text, "ok": True,
                               "depos": [[int(r["id"]), float(r["t"]), float(r["x"]), int(r["q"]),
                                          float(r["sigma_t"]), float(r["sigma_x"])] for r in d]}
            except Exception as e:  # OracleError carries the reference's what()
                cases[name] = {"text": text, "ok": False, "error": str(e).replace(str(path), "<path>")}
    (HERE / "golden_csv.json").write_text(json.dumps(
        {"gen": {"n": 64, "seed": 11, "grid": [48, 300, 12, 100, 5.0, 0.5]}, "cases": cases}, indent=1))
    print("wrote", HERE / "depos_ref.csv", HERE / "golden_csv.json")


def sigproc_fixtures(ref):
    """sigproc_chain (sigproc.cpp:104-118) and row_median (sigproc.cpp:80-102)
    known answers from the unmodified reference -> tests/golden/sigproc.npz."""
    rng = np.random.default_rng(2104)
    out = {}
    cases = [("c600", 16, 600, 3, 10, True), ("c735", 9, 735, 0, 9, True), ("c1", 4, 1, 1, 2, True),
             ("c64_real_filter", 6, 64, 2, 4, False)]
    for name, rows, cols, pad, nout, cfilt in cases:
        data = rng.normal(size=(rows, cols)) + 1j * rng.normal(size=(rows, cols))
        filt = (rng.normal(size=cols) + 1j * rng.normal(size=cols)) if cfilt else rng.normal(size=cols) + 0j
        block, med, mri, _ = ref.sigproc_chain(data, filt, pad, nout)
        out.update({f"{name}_data": data, f"{name}_filter": filt, f"{name}_block": block, f"{name}_medians": med,
                    f"{name}_meta": np.array([pad, nout, mri])})
    # Hermitian rows: forward DFT of real signals, identity filter (SPEC sigproc AC9)
    sig = rng.normal(size=(12, 6000))
    spec = np.fft.fft(sig, axis=1)
    block, med, mri, _ = ref.sigproc_chain(spec, np.ones(6000), 2, 8)
    out.update({"herm_signal": sig, "herm_block": block, "herm_medians": med, "herm_meta": np.array([2, 8, mri])})
    # row_median on ties, signed zeros, odd / even lengths
    med_rows = [np.array([3.0, 1.0, 2.0]), np.array([1.0, 2.0, 3.0, 4.0]), np.array([0.0, -0.0, 0.0, -0.0]),
                np.array([5.0] * 7), np.array([2.0, 2.0, 1.0, 1.0, 3.0, 3.0]), rng.normal(size=10000),
                rng.integers(-3, 4, size=1001).astype(np.float64), np.array([-1e300, 1e-300, -0.0, 7.0, 1e300])]
    for i, v in enumerate(med_rows):
        out[f"median{i}_in"] = v
        out[f"median{i}_out"] = np.array([ref.row_median(v), ref.row_median(v, by_sort=True)])
    np.savez_compressed(HERE / "sigproc.npz", **out)
    print("wrote", HERE / "sigproc.npz")


def main():
    build_ref()
    ref = Reference()
    csv_fixtures(ref)
    sigproc_fixtures(ref)
    if "--aux-only" in sys.argv:
        return
    gold = {}

    # Philox4x32-10 KATs (Random123)
    gold["philox_kat"] = [
        {"ctr": [0, 0, 0, 0], "key": [0, 0], "out": ref.philox([0, 0, 0, 0], [0, 0]).tolist()},
        {"ctr": [0, 0, 0, 0], "key": [12345, 0], "out": ref.philox([0, 0, 0, 0], [12345, 0]).tolist()},
        {"ctr": [7, 3, 1, 0], "key": [0xDEADBEEF, 0x1234], "out": ref.philox([7, 3, 1, 0], [0xDEADBEEF, 0x1234]).tolist()},
    ]
    # substream / philox draws (rng.cpp:51-76, rng.hpp:72-98; PhiloxSource in ref_harness.cpp)
    draws = []
    for mode in (0, 1):
        for sid in (0, 1, 7, (1 << 40) + 3):
            draws.append({"mode": mode, "seed": 12345, "id": sid,
                          "uniform": ref.draws(mode, 0, 12345, sid, 8).tolist(),
                          "normal": ref.draws(mode, 1, 12345, sid, 8).tolist()})
    gold["draws"] = draws
    # binomial (rng.cpp:174-193), including the lgamma-seeded walk
    gold["binomial"] = [
        {"n": n, "p": p, "seed": 7, "id": 3, "k": ref.binomials(n, p, 7, 3, 16).tolist()}
        for n, p in [(20, 0.3), (100, 0.05), (5000, 0.9), (5927, 0.11813274317501754), (1, 0.5), (57, 0.0), (57, 1.0)]
    ]
    # footprints and patches (core.cpp:25-41, rasterize.cpp:44-120)
    g = make_grid(48, 300, 12, 100, 5.0, 0.5)
    gspec = {"n_wires": 48, "n_ticks": 300, "pad_wires": 12, "pad_ticks": 100, "pitch": 5.0, "tick": 0.5}
    gold["grid_small"] = gspec
    ed = edge_depos()
    gold["edge_depos"] = {k: ed[k].tolist() for k in ed.dtype.names}
    gold["map_depo"] = [ref.map_depo(g, ed[i]).tolist() for i in range(len(ed))]
    patches = []
    for i in range(len(ed)):
        p = ref.sample_patch(g, ed[i])
        patches.append({k: (v.ravel().tolist() if isinstance(v, np.ndarray) else v) for k, v in p.items()})
    gold["sample_patch"] = patches
    # SPEC.md:60 example: tick 1 us, pitch 5 mm, origins 0 -> centre (wire 5, tick 10) (+pads)
    g1 = make_grid(100, 100, 0, 0, 5.0, 1.0)
    d1 = np.zeros(1, dtype=DEPO_DTYPE)
    d1["t"], d1["x"], d1["sigma_t"], d1["sigma_x"] = 10.2, 25.6, 3.3, 1.0
    gold["map_depo_spec"] = ref.map_depo(g1, d1[0]).tolist()
    # drift (rasterize.cpp:22-42); dx = 100 mm -> sigma_x' = 1.0488 mm
    d2 = np.zeros(1, dtype=DEPO_DTYPE)
    d2["x"], d2["t"] = 100.0, 5.0
    dd = ref.drift(d2, Drift(0.0, 1.6, 0.0068, 0.0088))
    gold["drift_spec"] = {k: float(dd[k][0]) for k in ("t", "x", "sigma_t", "sigma_x")}

    # a small full run: gen_depos + run_simulation (substream, pool) + fluct-off charge + convolve
    depos = ref.gen_depos(1500, 7, g)
    run = ref.run_simulation(g, make_response(), depos, workers=1)
    pool = ref.run_simulation(g, make_response(), depos, rng_mode=1, workers=1)
    phil, _ = ref.charge_fluct_philox(g, depos, seed=12345)
    s_off, clipped_off = ref.charge_fluct_off(g, depos)
    arrays = {
        "small_depos": depos.view(np.uint8),
        "small_charge_substream": run["charge"],
        "small_adc_substream": run["adc"],
        "small_charge_pool": pool["charge"],
        "small_charge_philox": phil,
        "small_charge_off": s_off,
    }
    for name, r in [("collection", make_response()), ("induction", make_response("induction")),
                    ("ww3", make_response("collection", wire_weights=(0.25, 1.0, 0.25)))]:
        arrays[f"small_m_off_{name}"] = ref.convolve_real(g, r, s_off)
        arrays[f"small_m_on_{name}"] = ref.convolve_int(g, r, run["charge"])
        rb = ref.build_response(g, r)
        gold[f"support_{name}"] = [rb["support_ticks"], rb["support_wires"]]
    gold["small_clipped_off"] = clipped_off
    gold["small_clipped_substream"] = run["clipped_charge"]
    noisy, adc = ref.noise_digitize(g, arrays["small_m_off_collection"], noise_mode=1, sigma=2.0, seed=12345)
    arrays["small_noisy_white"] = noisy
    arrays["small_adc_white"] = adc

    # C1 survey anchors: gen_depos(10000, seed 7) on 480 x 6000
    gc1 = make_grid(480, 6000)
    dc1 = ref.gen_depos(10000, 7, gc1)
    sub = ref.run_simulation(gc1, make_response(), dc1, workers=8)
    poolc1 = ref.run_simulation(gc1, make_response(), dc1, rng_mode=1, workers=8)
    philc1, _ = ref.charge_fluct_philox(gc1, dc1, seed=12345)
    offc1, _ = ref.charge_fluct_off(gc1, dc1)
    gold["c1"] = {
        "depos_fnv1a": fnv1a64(dc1),
        "charge_substream_fnv1a": fnv1a64(sub["charge"]), "charge_substream_sum": int(sub["charge"].sum()),
        "charge_pool_fnv1a": fnv1a64(poolc1["charge"]),
        "charge_philox_fnv1a": fnv1a64(philc1), "charge_philox_sum": int(philc1.sum()),
        "charge_off_sum": float(offc1.sum()), "clipped": int(sub["clipped_charge"]),
    }
    (HERE / "golden.json").write_text(json.dumps(gold, indent=1))
    np.savez_compressed(HERE / "golden_arrays.npz", **arrays)
    print("wrote", HERE / "golden.json", HERE / "golden_arrays.npz")


if __name__ == "__main__":
    main()
