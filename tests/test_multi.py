"""Multi-process host logic on CPU (gloo, world_size 2): the unit sharding
covers every (face, plane) exactly once, balances cost, and the union of the
per-rank results equals the single-process result (placement invariance).
The per-unit compute here is the CPU oracle standing in for the device."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_08265_b200.sharding import events_for_rank, protodune_units, shard_units, unit_cost


def test_shard_units_cover_and_balance():
    units = protodune_units()
    costs = [unit_cost(w, t, 5000) for _, _, w, t in units]
    for world in (1, 2, 4, 8):
        owned = shard_units(costs, world)
        flat = sorted(i for o in owned for i in o)
        assert flat == list(range(len(units)))
        loads = [sum(costs[i] for i in o) for o in owned]
        assert max(loads) <= sum(costs) / world + max(costs)  # LPT bound
    assert events_for_rank(64, 3, 8) == list(range(3, 64, 8))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _small_units():
    from oracle.oracle import make_grid
    grids = [make_grid(24 + 8 * i, 300, 6, 100, 5.0, 0.5) for i in range(5)]
    return grids


def _unit_result(i):
    from oracle.oracle import Oracle, make_response
    from paper_2104_08265_b200.api import GridSpec
    from paper_2104_08265_b200.workloads import line_tracks
    o = Oracle()
    g = _small_units()[i]
    gs = GridSpec(int(g.n_wires), int(g.n_ticks), int(g.pad_wires), int(g.pad_ticks), g.pitch, g.tick)
    d = line_tracks(120, gs, seed=100 + i)
    s, _ = o.charge_fluct_on(g, d, rng_mode=1, seed=77)  # keyed by (seed, depo id): placement-invariant
    return o.convolve(g, make_response("induction" if i % 2 else "collection"), s.astype(np.float64))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grids = _small_units()
    costs = [unit_cost(int(g.n_wires + 2 * g.pad_wires), int(g.n_ticks + 2 * g.pad_ticks), 120) for g in grids]
    mine = shard_units(costs, world)[rank]
    local = {i: _unit_result(i) for i in mine}
    gathered = [None] * world
    dist.all_gather_object(gathered, local)  # final frame gather (not on the hot path)
    if rank == 0:
        merged = {}
        for part in gathered:
            assert not set(part) & set(merged)
            merged.update(part)
        np.save(out, np.array([merged[i] for i in range(len(grids))], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_union_equals_single(tmp_path):
    out = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    merged = np.load(out, allow_pickle=True)
    for i in range(len(_small_units())):
        np.testing.assert_array_equal(merged[i], _unit_result(i))


def test_cost_model_matches_c_abi():
    """The Python sharding cost model is the C ABI's (ws_multi_cost, host-only)."""
    from paper_2104_08265_b200 import _lib
    lib = _lib.load()
    for w, t, n in ((2600, 9800, 100_000), (1000, 6200, 0), (680, 6200, 10_000)):
        assert lib.ws_multi_cost(w * t, n) == unit_cost(w, t, n)


def test_bench_rank_device_mapping(monkeypatch):
    """bench.py's rank -> device mapping: LOCAL_RANK as is (one GPU per rank),
    or modulo the visible devices in the shared-GPU test mode (a path check on
    a box with fewer GPUs than ranks; never a reported number)."""
    import importlib
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    bench = importlib.import_module("bench")
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("LOCAL_RANK", "3")
    monkeypatch.delenv("WS_BENCH_SHARED_GPU", raising=False)
    assert bench.dist_setup() == (4, 3, 3)
    monkeypatch.setenv("WS_BENCH_SHARED_GPU", "1")
    import torch
    n = max(1, torch.cuda.device_count())
    assert bench.dist_setup() == (4, 3, 3 % n)
