"""Shared test helpers: parity metrics and small configs."""
import numpy as np

from oracle.oracle import make_grid, make_response


def relL2_per_channel(m_gpu, m_ref, mask=None):
    """max over channels (padded wire rows) of ||M_gpu - M_ref|| / ||M_ref||,
    over rows whose reference row is non-zero (the oracle's direct convolution
    leaves signal-free rows exactly zero)."""
    m_gpu = np.asarray(m_gpu, dtype=np.float64)
    m_ref = np.asarray(m_ref, dtype=np.float64)
    num = np.sqrt(((m_gpu - m_ref) ** 2).sum(axis=1))
    den = np.sqrt((m_ref ** 2).sum(axis=1))
    if mask is None:
        mask = den > 0
    if not mask.any():
        return 0.0
    return float((num[mask] / den[mask]).max())


def oracle_grid(g):
    """oracle Grid struct from a paper_2104_08265_b200.GridSpec"""
    return make_grid(g.n_wires, g.n_ticks, g.pad_wires, g.pad_ticks, g.pitch, g.tick, g.origin_x, g.origin_t)


def oracle_response(r):
    return make_response(r.plane_kind, r.field_sigma_t, r.shaper_peaking, r.shaper_order, r.gain,
                         tuple(r.wire_weights))
