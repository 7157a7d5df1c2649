"""Placement of independent work units across GPUs.

Every (anode face, plane) of an event, and every event, is an independent
run_simulation-equivalent: no data crosses units, so ranks never exchange
data on the hot path. Work is balanced greedily by a cost model; the results
are placement-invariant because the fluctuation streams are keyed by
(seed, depo id) and the scatter is integer (bitwise reproducible).
"""
from __future__ import annotations

from typing import Sequence


DEPO_COST = 900.0  # cells-equivalent of one depo on one plane (ws_multi_cost in csrc/ws_multi.cu)


def unit_cost(padded_wires: int, padded_ticks: int, n_depos: int) -> float:
    """Device-time model of one plane run, the same as the C ABI's
    ws_multi_cost: the time-domain path (k_direct) writes every cell once and
    adds each depo's response profile (~12 wire rows x ~130 taps) to its rows;
    fitted to the C5 sweep (1k-1M depos per MicroBooNE event, round 2: 0.9-1.3
    ns per depo-plane vs 1.0 ps per cell): cost = cells + 900 x depos."""
    return float(padded_wires) * padded_ticks + DEPO_COST * n_depos


def shard_units(costs: Sequence[float], world: int) -> list[list[int]]:
    """Longest-processing-time-first greedy: returns, per rank, the unit indices
    it owns. Deterministic (ties broken by unit index)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    loads = [0.0] * world
    owned: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda k: (-costs[k], k)):
        r = min(range(world), key=lambda q: (loads[q], q))
        owned[r].append(i)
        loads[r] += costs[i]
    for o in owned:
        o.sort()
    return owned


def events_for_rank(n_events: int, rank: int, world: int) -> list[int]:
    """Round-robin event sharding (configs[4]: 64 events over 8 GPUs)."""
    return list(range(rank, n_events, world))


def protodune_units(n_faces: int = 12, wires=(800, 800, 480), n_ticks: int = 6000, pad: int = 100):
    """(face, plane, padded_wires, padded_ticks) of a ProtoDUNE-SP event (configs[3]):
    12 faces x U/V/W with 800/800/480 channels x 6000 ticks (domain numbers, not
    from the reference)."""
    return [(f, p, w + 2 * pad, n_ticks + 2 * pad) for f in range(n_faces) for p, w in enumerate(wires)]
