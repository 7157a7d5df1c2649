"""ctypes binding of the C ABI in include/wiresim_gpu.h (libwsgpu.so, built in-tree).

There is deliberately no fallback: if the CUDA library is missing or no sm_100
device is usable, calls raise ``WsError`` instead of computing anything on the
CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libwsgpu.so"

WS_OK, WS_EINVAL, WS_ERANGE, WS_EDOMAIN, WS_ERUNTIME, WS_ECUDA, WS_ENOMEM = range(7)
WS_INDUCTION, WS_COLLECTION = 0, 1
WS_RNG_SUBSTREAM, WS_RNG_PHILOX = 0, 1
WS_CHARGE_F32, WS_CHARGE_U32, WS_CHARGE_I64 = 0, 1, 2

# ws_depo == wiresim::Depo (core.hpp:63-70)
DEPO_DTYPE = np.dtype(
    [("id", "<i8"), ("t", "<f8"), ("x", "<f8"), ("q", "<i8"), ("sigma_t", "<f8"), ("sigma_x", "<f8")]
)


class WsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[ws status {code}] {msg}")
        self.code = code


class GridSpecC(C.Structure):
    _fields_ = [
        ("n_wires", C.c_uint64), ("n_ticks", C.c_uint64), ("pad_wires", C.c_uint64), ("pad_ticks", C.c_uint64),
        ("pitch", C.c_double), ("tick", C.c_double), ("origin_x", C.c_double), ("origin_t", C.c_double),
    ]


class ResponseC(C.Structure):
    _fields_ = [
        ("plane_kind", C.c_int32), ("shaper_order", C.c_int32), ("field_sigma_t", C.c_double),
        ("shaper_peaking", C.c_double), ("gain", C.c_double), ("wire_weights", C.POINTER(C.c_double)),
        ("n_wire_weights", C.c_uint64),
    ]


class DriftC(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("reserved", C.c_int32), ("response_plane_x", C.c_double),
                ("drift_speed", C.c_double), ("diffusion_long", C.c_double), ("diffusion_tran", C.c_double)]


class SimOptionsC(C.Structure):
    _fields_ = [("fluctuate", C.c_int32), ("approx", C.c_int32), ("rng_mode", C.c_int32), ("charge_type", C.c_int32),
                ("seed", C.c_uint64), ("drift", DriftC)]


class NoiseModelC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("rng_mode", C.c_int32), ("sigma", C.c_double), ("seed", C.c_uint64),
                ("amplitude_spectrum", C.c_void_p), ("n_amplitude", C.c_uint64)]


class AdcConfigC(C.Structure):
    _fields_ = [("scale", C.c_double), ("offset", C.c_double), ("bits", C.c_int32), ("reserved", C.c_int32)]


WS_FRAME_F32, WS_FRAME_F64 = 0, 1
WS_ADC_I32, WS_ADC_U16 = 0, 1
WS_NOISE_OFF, WS_NOISE_WHITE, WS_NOISE_SPECTRUM = 0, 1, 2


class ReadoutC(C.Structure):
    _fields_ = [("noise", NoiseModelC), ("adc", AdcConfigC), ("frame_type", C.c_int32), ("adc_type", C.c_int32)]


class SignalBatchC(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_uint64), ("cols", C.c_uint64), ("pad_rows", C.c_uint64),
                ("out_rows", C.c_uint64)]


class TimingC(C.Structure):
    _fields_ = [("prepare_ms", C.c_float), ("fluctuate_ms", C.c_float), ("bin_ms", C.c_float),
                ("convolve_ms", C.c_float), ("total_ms", C.c_float), ("direct_planes", C.c_int32),
                ("clipped_patches", C.c_int64), ("clipped_charge", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PlaneInfoC(C.Structure):
    _fields_ = [("padded_wires", C.c_uint64), ("padded_ticks", C.c_uint64), ("fft_length", C.c_uint64),
                ("folded", C.c_int32), ("n_radix_passes", C.c_int32), ("support_ticks", C.c_int64),
                ("support_wires", C.c_int64), ("lo_lag", C.c_int64), ("n_lags", C.c_int64),
                ("impacts_per_pitch", C.c_int32), ("n_response_classes", C.c_int32)]


# exported symbols (name -> (restype, argtypes)); every one is declared in include/*.h
_P = C.c_void_p
SIGNATURES = {
    "ws_last_error": (C.c_char_p, []),
    "ws_abi_version": (C.c_int, []),
    "ws_ctx_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    "ws_ctx_destroy": (C.c_int, [_P]),
    "ws_ctx_synchronize": (C.c_int, [_P]),
    "ws_ctx_stream": (_P, [_P]),
    "ws_ctx_launch_count": (C.c_uint64, [_P]),
    "ws_ctx_set_conv_path": (C.c_int, [_P, C.c_int]),
    "ws_ctx_set_direct_kappa": (C.c_int, [_P, C.c_double]),
    "ws_plane_create": (C.c_int, [_P, C.POINTER(GridSpecC), C.POINTER(ResponseC), C.c_double, C.POINTER(_P)]),
    "ws_plane_create_impacts": (C.c_int, [_P, C.POINTER(GridSpecC), _P, C.c_uint32, C.c_double, C.POINTER(_P)]),
    "ws_plane_destroy": (C.c_int, [_P]),
    "ws_plane_get_info": (C.c_int, [_P, C.POINTER(PlaneInfoC)]),
    "ws_plane_get_kernel": (C.c_int, [_P, _P, C.c_uint64]),
    "ws_rasterize_device": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(SimOptionsC), _P, C.POINTER(TimingC)]),
    "ws_convolve_device": (C.c_int, [_P, _P, _P]),
    "ws_simulate_plane_device": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(SimOptionsC), _P, _P, C.POINTER(TimingC)]),
    "ws_simulate_plane": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(SimOptionsC), _P, _P, C.POINTER(TimingC)]),
    "ws_simulate_event_device": (C.c_int, [_P, C.c_uint32, _P, _P, _P, C.POINTER(SimOptionsC), _P,
                                           C.POINTER(TimingC)]),
    "ws_simulate_event": (C.c_int, [_P, C.c_uint32, _P, _P, _P, C.POINTER(SimOptionsC), _P, C.POINTER(TimingC)]),
    "ws_simulate_events": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P, _P, C.POINTER(SimOptionsC), _P,
                                     C.POINTER(TimingC)]),
    "ws_run_simulation": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(SimOptionsC), C.POINTER(ReadoutC), _P, _P, _P,
                                    C.POINTER(TimingC)]),
    "ws_run_simulation_device": (C.c_int, [_P, _P, C.c_uint64, C.POINTER(SimOptionsC), C.POINTER(ReadoutC), _P, _P,
                                           _P, C.POINTER(TimingC)]),
    "ws_run_event_device": (C.c_int, [_P, C.c_uint32, _P, _P, _P, C.POINTER(SimOptionsC), C.POINTER(ReadoutC), _P, _P,
                                      C.POINTER(TimingC)]),
    "ws_run_events": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, _P, _P, C.POINTER(SimOptionsC), C.POINTER(ReadoutC),
                                _P, _P, C.POINTER(TimingC)]),
    "ws_multi_create": (C.c_int, [C.c_uint32, _P, C.c_uint32, _P, _P, C.c_double, C.POINTER(_P)]),
    "ws_multi_destroy": (C.c_int, [_P]),
    "ws_multi_device_count": (C.c_uint32, [_P]),
    "ws_multi_context": (_P, [_P, C.c_uint32]),
    "ws_multi_plane": (_P, [_P, C.c_uint32, C.c_uint32]),
    "ws_multi_set_conv_path": (C.c_int, [_P, C.c_int]),
    "ws_multi_cost": (C.c_double, [C.c_uint64, C.c_uint64]),
    "ws_multi_run_events": (C.c_int, [_P, C.c_uint32, _P, _P, C.POINTER(SimOptionsC), C.POINTER(ReadoutC), _P, _P,
                                      _P, C.POINTER(TimingC)]),
    "ws_multi_run_units": (C.c_int, [_P, C.c_uint32, _P, _P, _P, C.POINTER(SimOptionsC), C.POINTER(ReadoutC), _P,
                                     _P, _P]),
    "ws_gen_depos_uniform":(C.c_int, [C.c_uint64, C.c_uint64, C.POINTER(GridSpecC), _P, _P]),
    "ws_noise_digitize_device": (C.c_int, [_P, _P, C.POINTER(NoiseModelC), C.c_double, C.c_double, C.c_int32, _P]),
    "ws_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(_P)]),
    "ws_host_free": (C.c_int, [_P]),
    "ws_sigproc_chain_device": (C.c_int, [_P, C.POINTER(SignalBatchC), _P, C.c_uint64, _P, _P,
                                          C.POINTER(C.c_double)]),
    "ws_sigproc_chain": (C.c_int, [_P, C.POINTER(SignalBatchC), _P, C.c_uint64, C.c_int, _P, _P,
                                   C.POINTER(C.c_double)]),
    "ws_row_medians_device": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64, _P]),
    "ws_sigproc_max_cols": (C.c_uint64, []),
    "ws_load_depos_csv": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_P), C.POINTER(C.c_uint64)]),
    "ws_free_depos": (C.c_int, [_P, C.c_int]),
    "ws_save_depos_csv": (C.c_int, [C.c_char_p, _P, C.c_uint64]),
}

_lib = None


def load() -> C.CDLL:
    """Load libwsgpu.so (raises if it has not been built: there is no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("WS_GPU_LIB", LIB_PATH))
    if not path.exists():
        raise WsError(WS_ECUDA, f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc != WS_OK:
        raise WsError(rc, load().ws_last_error().decode())
