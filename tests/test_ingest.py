"""Depo ingestion: the native CSV reader/writer of the
C ABI against the reference's load_depos / gen_depos (pipeline.cpp:226-294).

Fixtures from tests/golden/make_golden.py (unmodified reference): a file
written by gen_depos and the reference loader's verdict on edge-case files.
Host-only calls, so these run without a GPU.
"""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2104_08265_b200 import DEPO_DTYPE, GridSpec, WsError, gen_depos, load_depos, save_depos

GOLD = Path(__file__).resolve().parent / "golden"
CSV = json.loads((GOLD / "golden_csv.json").read_text())


def _grid():
    n_w, n_t, p_w, p_t, pitch, tick = CSV["gen"]["grid"]
    return GridSpec(n_wires=n_w, n_ticks=n_t, pad_wires=p_w, pad_ticks=p_t, pitch=pitch, tick=tick)


def test_load_reference_file_matches_generator():
    got = load_depos(GOLD / "depos_ref.csv")
    want = gen_depos(CSV["gen"]["n"], CSV["gen"]["seed"], _grid())
    assert got.dtype == DEPO_DTYPE and len(got) == CSV["gen"]["n"]
    assert got.tobytes() == want.tobytes()  # %.17g text is exact


def test_save_is_byte_identical_to_reference_writer(tmp_path):
    d = gen_depos(CSV["gen"]["n"], CSV["gen"]["seed"], _grid())
    out = tmp_path / "d.csv"
    save_depos(out, d)
    assert out.read_bytes() == (GOLD / "depos_ref.csv").read_bytes()


def test_round_trip_large(tmp_path):
    d = gen_depos(200_000, 5, GridSpec(n_wires=3456, n_ticks=9600))
    out = tmp_path / "big.csv"
    save_depos(out, d)
    assert load_depos(out).tobytes() == d.tobytes()


@pytest.mark.parametrize("name", sorted(CSV["cases"]))
def test_edge_cases_match_reference_loader(tmp_path, name):
    case = CSV["cases"][name]
    path = tmp_path / f"{name}.csv"
    path.write_bytes(case["text"].encode())
    if case["ok"]:
        got = load_depos(path)
        want = np.array([tuple(r) for r in case["depos"]], dtype=DEPO_DTYPE)
        assert got.tobytes() == want.tobytes()
    else:
        with pytest.raises(WsError) as ei:
            load_depos(path)
        assert str(ei.value).endswith(case["error"].replace("<path>", str(path)))


def test_missing_file_and_bad_ids(tmp_path):
    with pytest.raises(WsError, match="cannot open"):
        load_depos(tmp_path / "nope.csv")
    d = np.zeros(2, dtype=DEPO_DTYPE)
    d["id"] = [0, 5]
    with pytest.raises(WsError, match="row index"):
        save_depos(tmp_path / "x.csv", d)
