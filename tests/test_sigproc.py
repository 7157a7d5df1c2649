"""Signal-processing chain (sigproc.cpp:104-118, the
paper's Listing 1): filter -> inverse DFT along rows -> block cut -> medians.

Fixtures in tests/golden/sigproc.npz come from the unmodified reference
(tests/golden/make_golden.py). The CPU tests pin the oracle's restatement
(oracle/wsoracle.c) to them; the GPU tests check the sm_100a kernel
(csrc/ws_sigproc.cu) against the fixtures, the oracle at the paper's size
(960 x 6000) and numpy.

Tolerances: the chain is fp64 end to end; different FFT factorisations agree
to a few ulps of the row's peak, so blocks are compared at relL2 <= 1e-12
(SPEC's sigproc bound is 1e-9) and medians at <= 1e-12 x the row peak.
Medians of given values (row_median alone) are exact.
"""
from pathlib import Path

import numpy as np
import pytest

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "sigproc.npz")
CASES = ["c600", "c735", "c1", "c64_real_filter"]
N_MED = len([k for k in GOLD.files if k.startswith("median") and k.endswith("_in")])


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _case(name):
    pad, out, mri = GOLD[f"{name}_meta"]
    return GOLD[f"{name}_data"], GOLD[f"{name}_filter"], int(pad), int(out), float(mri)


# ---- oracle pinned to the reference (CPU) ----------------------------------

@pytest.mark.parametrize("name", CASES)
def test_oracle_chain_matches_reference(oracle, name):
    data, filt, pad, out, mri = _case(name)
    block, med, got_mri = oracle.sigproc_chain(data, filt, pad, out)
    assert block.shape == GOLD[f"{name}_block"].shape
    assert _rel(block, GOLD[f"{name}_block"]) <= 1e-13
    assert np.max(np.abs(med - GOLD[f"{name}_medians"])) <= 1e-13 * max(np.max(np.abs(block)), 1e-300)
    assert got_mri == pytest.approx(mri, rel=1e-9)


def test_oracle_hermitian_round_trip(oracle):
    sig = GOLD["herm_signal"]
    block, med, mri = oracle.sigproc_chain(np.fft.fft(sig, axis=1), np.ones(sig.shape[1]), 2, 8)
    assert _rel(block, GOLD["herm_block"]) <= 1e-13
    assert _rel(block, sig[2:10]) <= 1e-13


@pytest.mark.parametrize("i", range(N_MED))
def test_oracle_median_matches_reference(oracle, i):
    want = GOLD[f"median{i}_out"]
    assert want[0] == want[1]  # row_median == row_median_by_sort in the reference
    assert oracle.row_median(GOLD[f"median{i}_in"]) == want[0]


# ---- GPU ------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_gpu_chain_matches_reference(ctx, name):
    from paper_2104_08265_b200 import sigproc_chain
    data, filt, pad, out, mri = _case(name)
    if name == "c64_real_filter":
        filt = filt.real.copy()  # the double overload of apply_filter
    r = sigproc_chain(data, filt, pad, out, ctx=ctx)
    want = GOLD[f"{name}_block"]
    assert r.block.shape == want.shape
    assert _rel(r.block, want) <= 1e-12
    peak = max(np.max(np.abs(want)), 1e-300)
    assert np.max(np.abs(r.medians - GOLD[f"{name}_medians"])) <= 1e-12 * peak
    assert r.max_rel_imag == pytest.approx(mri, rel=1e-9)


@pytest.mark.gpu
def test_gpu_hermitian_round_trip(ctx):
    from paper_2104_08265_b200 import sigproc_chain
    sig = GOLD["herm_signal"]
    r = sigproc_chain(np.fft.fft(sig, axis=1), np.ones(sig.shape[1]), 2, 8, ctx=ctx)
    assert _rel(r.block, GOLD["herm_block"]) <= 1e-12
    assert _rel(r.block, sig[2:10]) <= 1e-12
    assert r.max_rel_imag < 1e-12
    assert np.max(np.abs(r.medians - GOLD["herm_medians"])) <= 1e-12 * np.max(np.abs(sig))


@pytest.mark.gpu
def test_gpu_paper_size_vs_oracle(ctx, oracle):
    """960 x 6000 (the paper's 800~960 signals x 6000 samples), complex filter,
    80 guard rows; several host-path chunks, block edges inside chunks."""
    from paper_2104_08265_b200 import sigproc_chain
    rng = np.random.default_rng(6000)
    data = rng.normal(size=(960, 6000)) + 1j * rng.normal(size=(960, 6000))
    filt = np.exp(-np.linspace(0, 4, 6000)) * np.exp(1j * rng.uniform(0, 2 * np.pi, 6000))
    r = sigproc_chain(data, filt, 80, 800, ctx=ctx)
    block, med, mri = oracle.sigproc_chain(data, filt, 80, 800)
    assert _rel(r.block, block) <= 1e-12
    row_peak = np.max(np.abs(block), axis=1)
    assert np.all(np.abs(r.medians - med) <= 1e-12 * row_peak)
    assert r.max_rel_imag == pytest.approx(mri, rel=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 7, 8, 12, 13, 60, 64, 343, 1000, 1024, 1144, 4096, 6000, 8192, 9600, 13312,
                               17, 97, 2 * 3 * 17, 1009, 6007])  # the last five: direct-DFT path
def test_gpu_lengths_vs_numpy(ctx, n):
    from paper_2104_08265_b200 import sigproc_chain
    rng = np.random.default_rng(n)
    rows = 5
    data = rng.normal(size=(rows, n)) + 1j * rng.normal(size=(rows, n))
    filt = rng.normal(size=n) + 1j * rng.normal(size=n)
    r = sigproc_chain(data, filt, 1, 3, ctx=ctx)
    want = np.fft.ifft(data * filt, axis=1)
    assert _rel(r.block, want.real[1:4]) <= 1e-13
    for i in range(3):
        assert abs(r.medians[i] - np.median(r.block[i])) <= 1e-15 * np.max(np.abs(r.block[i]))
    mri = np.max(np.abs(want.imag)) / np.max(np.abs(want.real))
    assert r.max_rel_imag == pytest.approx(mri, rel=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(N_MED))
def test_gpu_row_median_exact(ctx, i):
    import torch
    from paper_2104_08265_b200 import row_medians_device
    v = torch.from_numpy(GOLD[f"median{i}_in"].copy()).cuda().reshape(1, -1)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    row_medians_device(ctx, v, 1, v.shape[1], out)
    ctx.synchronize()
    assert out.item() == GOLD[f"median{i}_out"][0]


@pytest.mark.gpu
def test_gpu_row_medians_many(ctx):
    import torch
    from paper_2104_08265_b200 import row_medians_device
    rng = np.random.default_rng(5)
    for cols in (1, 2, 3, 999, 1000, 6000):
        m = rng.normal(size=(64, cols))
        m[::3] = np.round(m[::3])  # ties
        d = torch.from_numpy(m).cuda()
        out = torch.empty(64, dtype=torch.float64, device="cuda")
        row_medians_device(ctx, d, 64, cols, out)
        ctx.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), np.median(m, axis=1))


@pytest.mark.gpu
def test_gpu_device_path_equals_host_path(ctx):
    import torch
    from paper_2104_08265_b200 import sigproc_chain, sigproc_chain_device
    rng = np.random.default_rng(9)
    data = rng.normal(size=(300, 6000)) + 1j * rng.normal(size=(300, 6000))
    filt = rng.normal(size=6000) + 1j * rng.normal(size=6000)
    host = sigproc_chain(data, filt, 7, 250, ctx=ctx)
    dd = torch.from_numpy(data).cuda()
    fd = torch.from_numpy(filt).cuda()
    blk = torch.empty((250, 6000), dtype=torch.float64, device="cuda")
    med = torch.empty(250, dtype=torch.float64, device="cuda")
    mri = sigproc_chain_device(ctx, dd, 300, 6000, fd, blk, med, pad_rows=7, out_rows=250, residue=True)
    np.testing.assert_array_equal(blk.cpu().numpy(), host.block)
    np.testing.assert_array_equal(med.cpu().numpy(), host.medians)
    assert mri == host.max_rel_imag


@pytest.mark.gpu
def test_gpu_errors(ctx):
    from paper_2104_08265_b200 import WsError, sigproc_chain, sigproc_max_cols
    d = np.zeros((1, 9973), dtype=np.complex128)  # prime, beyond the direct path's shared-memory row
    with pytest.raises(WsError, match="prime factor > 13 and exceeds"):
        sigproc_chain(d, np.ones(9973), 0, 1, ctx=ctx)
    d = np.zeros((4, 16), dtype=np.complex128)
    with pytest.raises(WsError, match="filter length 15 does not match 16"):
        sigproc_chain(d, np.ones(15), 0, 4, ctx=ctx)
    with pytest.raises(WsError, match="pad_rows \\+ out_rows exceeds"):
        sigproc_chain(d, np.ones(16), 2, 3, ctx=ctx)
    n = sigproc_max_cols() + 64
    with pytest.raises(WsError, match="exceeds"):
        sigproc_chain(np.zeros((1, n), dtype=np.complex128), np.ones(n), 0, 1, ctx=ctx)
    r = sigproc_chain(d, np.ones(16), 4, 0, ctx=ctx)  # no block rows
    assert r.block.shape == (0, 16)
