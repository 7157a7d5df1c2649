"""Synthetic depo workloads (inputs only; never part of a timed region).

* ``line_tracks``       2D line-track depos on one plane.
* ``microboone_event``  one MicroBooNE-scale event: 3D straight tracks in the
  TPC volume projected onto U/V (+-60 deg induction) and W (collection)
  planes of 2400/2400/3456 wires x 9600 ticks (BASELINE.json configs[1]).
  Wire pitch 3 mm (MicroBooNE's), tick 0.5 us, pad 100 wires / 100 ticks.
  Charge and widths follow the reference's DepoGenRanges defaults
  (pipeline.hpp:83-87): q ~ U[1000, 10000] e-, sigma_t ~ U[0.5, 1.5] us,
  sigma_x ~ U[2.5, 7.5] mm.
"""
from __future__ import annotations

import numpy as np

from ._lib import DEPO_DTYPE
from .api import GridSpec, ResponseParams

Q_RANGE = (1000, 10000)
SIGMA_T = (0.5, 1.5)
SIGMA_X = (2.5, 7.5)


def _fill(out, rng, t, x):
    n = len(out)
    out["id"] = np.arange(n, dtype=np.int64)
    out["t"] = t
    out["x"] = x
    out["q"] = rng.integers(Q_RANGE[0], Q_RANGE[1] + 1, size=n)
    out["sigma_t"] = rng.uniform(*SIGMA_T, size=n)
    out["sigma_x"] = rng.uniform(*SIGMA_X, size=n)
    return out


def line_tracks(n: int, grid: GridSpec, seed: int = 1, n_tracks: int | None = None) -> np.ndarray:
    """n depos spread evenly along K random straight tracks inside the active grid."""
    rng = np.random.default_rng(seed)
    k = n_tracks or max(1, n // 250)
    t_span = grid.n_ticks * grid.tick
    x_span = grid.n_wires * grid.pitch
    track = np.repeat(np.arange(k), int(np.ceil(n / k)))[:n]
    a = rng.uniform(0, 1, size=(k, 2))
    b = rng.uniform(0, 1, size=(k, 2))
    s = rng.uniform(0, 1, size=n)
    p = a[track] + (b[track] - a[track]) * s[:, None]
    out = np.zeros(n, dtype=DEPO_DTYPE)
    return _fill(out, rng, grid.origin_t + p[:, 0] * t_span, grid.origin_x + p[:, 1] * x_span)


MICROBOONE_PLANES = (
    # name, wires, kind, (cos, sin) of the wire-coordinate axis in (z, y)
    ("U", 2400, "induction", (0.5, 0.8660254037844386)),
    ("V", 2400, "induction", (0.5, -0.8660254037844386)),
    ("W", 3456, "collection", (1.0, 0.0)),
)
MICROBOONE_PITCH = 3.0
MICROBOONE_TICKS = 9600
MICROBOONE_Y = 2330.0   # mm, TPC height
MICROBOONE_Z = 10368.0  # mm, TPC length (3456 x 3 mm)


def microboone_grids():
    grids, responses = [], []
    for _, wires, kind, _ in MICROBOONE_PLANES:
        grids.append(GridSpec(n_wires=wires, n_ticks=MICROBOONE_TICKS, pad_wires=100, pad_ticks=100,
                              pitch=MICROBOONE_PITCH, tick=0.5))
        responses.append(ResponseParams(plane_kind=kind))
    return grids, responses


def microboone_event(n: int = 100_000, seed: int = 1, n_tracks: int | None = None):
    """One event: n depos on straight 3D tracks, projected to the U, V, W planes.

    Returns a list of three depo arrays (same ids / charges / widths, plane
    coordinate x differs)."""
    rng = np.random.default_rng(seed)
    k = n_tracks or max(1, n // 400)
    t_span = MICROBOONE_TICKS * 0.5
    track = np.repeat(np.arange(k), int(np.ceil(n / k)))[:n]
    lo = np.array([0.02, 0.02, 0.02])
    hi = np.array([0.98, 0.98, 0.98])
    a = rng.uniform(lo, hi, size=(k, 3))  # (t, y, z) in unit box
    b = a + rng.normal(0, 0.15, size=(k, 3))
    b = np.clip(b, lo, hi)
    s = rng.uniform(0, 1, size=n)
    p = a[track] + (b[track] - a[track]) * s[:, None]
    t = p[:, 0] * t_span
    y = p[:, 1] * MICROBOONE_Y
    z = p[:, 2] * MICROBOONE_Z
    base = np.zeros(n, dtype=DEPO_DTYPE)
    _fill(base, rng, t, np.zeros(n))
    out = []
    for _, wires, _, (cz, sy) in MICROBOONE_PLANES:
        d = base.copy()
        coord = cz * z + sy * y
        if sy < 0:
            coord = coord - sy * MICROBOONE_Y  # shift V into [0, span)
        d["x"] = np.clip(coord, 0.0, wires * MICROBOONE_PITCH - 1e-6)
        out.append(d)
    return out


PROTODUNE_WIRES = (800, 800, 480)   # U, V, W channels per anode face (ProtoDUNE-SP, domain numbers)
PROTODUNE_KINDS = ("induction", "induction", "collection")
PROTODUNE_FACES = 12                # 6 APAs x 2 faces


def protodune_specs():
    """(GridSpec, ResponseParams) of the three plane kinds of one anode face
    (BASELINE.json configs[3]): 800/800/480 wires x 6000 ticks, pad 100/100,
    pitch 5 mm; induction planes with +-1 wire coupling."""
    specs = []
    for wires, kind in zip(PROTODUNE_WIRES, PROTODUNE_KINDS):
        g = GridSpec(n_wires=wires, n_ticks=6000, pad_wires=100, pad_ticks=100, pitch=5.0, tick=0.5)
        r = ResponseParams(plane_kind=kind, wire_weights=(0.1, 1.0, 0.1) if kind == "induction" else (1.0,))
        specs.append((g, r))
    return specs


def protodune_event(n_per_unit: int = 20_000, seed: int = 1):
    """A 6-APA event as 36 independent (face, plane) units: returns
    (plane_of[36], depos[36]); unit u = face u // 3, plane kind u % 3; each
    unit's depos lie on line tracks across its face (n_per_unit each)."""
    specs = protodune_specs()
    plane_of, depos = [], []
    for f in range(PROTODUNE_FACES):
        for p in range(3):
            plane_of.append(p)
            depos.append(line_tracks(n_per_unit, specs[p][0], seed=1000 * seed + 3 * f + p))
    return plane_of, depos
