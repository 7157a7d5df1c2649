"""B200-native Wire-Cell signal-simulation hot path (arXiv 2104.08265).

rasterize -> scatter-add -> FFT convolution behind the C ABI in
include/wiresim_gpu.h; this package is the Python mirror of the reference's
C++ interface (see api.py) plus the synthetic workloads used by bench.py.
"""
from ._lib import DEPO_DTYPE, WsError  # noqa: F401
from .api import (  # noqa: F401
    AdcConfig,
    Context,
    Multi,
    NoiseModel,
    RunResult,
    run_events,
    DriftParams,
    GridSpec,
    Plane,
    ResponseParams,
    RngConfig,
    SimConfig,
    SimResult,
    gen_depos,
    load_depos,
    run_simulation,
    row_medians_device,
    sigproc_chain,
    sigproc_chain_device,
    sigproc_max_cols,
    ChainResult,
    save_depos,
    simulate_event,
    simulate_event_device,
    simulate_events,
)
