"""Host-side mirror of the reference's C++ interface for the hot path.

Types and field names follow /root/reference/proj/include/wiresim:
``GridSpec`` (core.hpp:40-58), ``ResponseParams`` (spectral.hpp:18-26),
``DriftParams`` (rasterize.hpp:16-23), ``RngConfig``/``SimConfig``
(pipeline.hpp:24-50), ``Depo`` arrays (core.hpp:63-70, as a numpy structured
array with the same 48-byte layout), and ``run_simulation``-shaped entry points
(pipeline.hpp:104) that stop at the pre-noise frame M = IFT(R . FT(S)) — the
raster -> scatter -> convolve section this library replaces.

Everything runs through libwsgpu.so (include/wiresim_gpu.h); there is no CPU
fallback. Errors raise ``WsError`` carrying the reference exception category
(WS_EINVAL ~ std::invalid_argument, WS_EDOMAIN ~ std::domain_error, ...).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import DEPO_DTYPE, WsError, check


@dataclass
class GridSpec:
    n_wires: int = 1000
    n_ticks: int = 6000
    pad_wires: int = 100
    pad_ticks: int = 100
    pitch: float = 5.0
    tick: float = 0.5
    origin_x: float = 0.0
    origin_t: float = 0.0

    def padded_wires(self) -> int:
        return self.n_wires + 2 * self.pad_wires

    def padded_ticks(self) -> int:
        return self.n_ticks + 2 * self.pad_ticks

    def to_c(self) -> _lib.GridSpecC:
        return _lib.GridSpecC(self.n_wires, self.n_ticks, self.pad_wires, self.pad_ticks, self.pitch, self.tick,
                              self.origin_x, self.origin_t)


@dataclass
class ResponseParams:
    plane_kind: str = "collection"  # "induction" | "collection"
    field_sigma_t: float = 1.0
    shaper_peaking: float = 2.0
    shaper_order: int = 2
    gain: float = 14.0
    wire_weights: Sequence[float] = (1.0,)

    def to_c(self):
        ww = np.ascontiguousarray(np.asarray(self.wire_weights, dtype=np.float64))
        r = _lib.ResponseC(_lib.WS_COLLECTION if self.plane_kind == "collection" else _lib.WS_INDUCTION,
                           self.shaper_order, self.field_sigma_t, self.shaper_peaking, self.gain,
                           ww.ctypes.data_as(C.POINTER(C.c_double)), ww.size)
        return r, ww


@dataclass
class DriftParams:
    response_plane_x: float = 0.0
    drift_speed: float = 1.6
    diffusion_long: float = 0.0068
    diffusion_tran: float = 0.0088
    enabled: bool = False


@dataclass
class RngConfig:
    mode: str = "substream"  # "substream" (reference xoshiro) | "philox" (shared counter stream)
    seed: int = 12345


@dataclass
class NoiseModel:
    """NoiseModel (spectral.hpp:51-55). rng: the per-wire stream, "substream"
    (the reference's, sequential per wire: a second kernel) or "philox"
    (counter-based: fused into the convolution's frame stores)."""
    mode: str = "off"  # "off" | "white" | "spectrum"
    sigma: float = 0.0
    amplitude_spectrum: Sequence[float] | None = None
    rng: str = "substream"


@dataclass
class AdcConfig:
    """AdcConfig (pipeline.hpp:30-34)."""
    scale: float = 1.0
    offset: float = 2048.0
    bits: int = 12


@dataclass
class SimConfig:
    grid: GridSpec = field(default_factory=GridSpec)
    drift: DriftParams = field(default_factory=DriftParams)
    response: ResponseParams = field(default_factory=ResponseParams)
    noise: NoiseModel = field(default_factory=NoiseModel)
    n_sigma: float = 3.0
    rng: RngConfig = field(default_factory=RngConfig)
    adc: AdcConfig = field(default_factory=AdcConfig)
    fluctuate: bool = True       # the reference always fluctuates (rasterize.cpp:182-202)
    approx: bool = False         # fluctuate_approx sampler (rasterize.cpp:159-170)

    def readout(self, adc_type: str = "i32", frame_type: str = "f32"):
        """(ReadoutC, keep-alive) for the ws_run_* entry points; the noise
        seed is rng.seed, as run_simulation passes it (pipeline.cpp:421)."""
        n = self.noise
        amp = None
        if n.mode == "spectrum":
            amp = np.ascontiguousarray(n.amplitude_spectrum, dtype=np.float64)
        mode = {"off": _lib.WS_NOISE_OFF, "white": _lib.WS_NOISE_WHITE, "spectrum": _lib.WS_NOISE_SPECTRUM}[n.mode]
        nm = _lib.NoiseModelC(mode, _lib.WS_RNG_PHILOX if n.rng == "philox" else _lib.WS_RNG_SUBSTREAM,
                              float(n.sigma), int(self.rng.seed), amp.ctypes.data if amp is not None else None,
                              amp.size if amp is not None else 0)
        r = _lib.ReadoutC(nm, _lib.AdcConfigC(self.adc.scale, self.adc.offset, self.adc.bits, 0),
                          _lib.WS_FRAME_F64 if frame_type == "f64" else _lib.WS_FRAME_F32,
                          _lib.WS_ADC_U16 if adc_type == "u16" else _lib.WS_ADC_I32)
        return r, amp

    def options(self, charge_type: str = "f32") -> _lib.SimOptionsC:
        """ws_sim_options; charge_type: with fluctuation, the charge outputs'
        type: "f32", "u32" (exact counts) or "i64" (the reference's int64)."""
        d = self.drift
        return _lib.SimOptionsC(
            int(self.fluctuate), int(self.approx),
            _lib.WS_RNG_PHILOX if self.rng.mode == "philox" else _lib.WS_RNG_SUBSTREAM, {"f32": 0, "u32": 1, "i64": 2}[charge_type],
            self.rng.seed,
            _lib.DriftC(int(d.enabled), 0, d.response_plane_x, d.drift_speed, d.diffusion_long, d.diffusion_tran))


def as_depos(depos) -> np.ndarray:
    a = np.ascontiguousarray(depos)
    if a.dtype != DEPO_DTYPE:
        a = np.ascontiguousarray(a.astype(DEPO_DTYPE))
    return a


class Context:
    """One device + stream + workspace (ws_ctx)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = _lib.load()
        h = C.c_void_p()
        check(self.lib.ws_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.handle = h
        self.device = device
        self._planes = weakref.WeakSet()  # closed before the context (a plane lives on its context)

    def synchronize(self):
        check(self.lib.ws_ctx_synchronize(self.handle))

    @property
    def stream(self) -> int:
        return self.lib.ws_ctx_stream(self.handle) or 0

    @property
    def launch_count(self) -> int:
        return int(self.lib.ws_ctx_launch_count(self.handle))

    CONV_PATHS = {"auto": 0, "fft": 1, "direct": 2}

    def set_conv_path(self, path: str):
        """Fluctuation-off convolution kernel: "auto" (per band of wire rows,
        the cheaper of time-domain accumulation and row FFT), "fft", "direct"."""
        check(self.lib.ws_ctx_set_conv_path(self.handle, self.CONV_PATHS[path]))

    def set_direct_kappa(self, kappa: float):
        """"auto" routing threshold (time-domain work per band <= kappa x transform length)."""
        check(self.lib.ws_ctx_set_direct_kappa(self.handle, float(kappa)))

    def close(self):
        if self.handle:
            for p in list(self._planes):
                p.close()
            self.lib.ws_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plane:
    """Geometry + response, precomputed on the device (ws_plane)."""

    def __init__(self, ctx: Context, grid: GridSpec, response: ResponseParams | Sequence[ResponseParams],
                 n_sigma: float = 3.0, impacts_per_pitch: int = 1):
        """response: one ResponseParams, or (impact positions,
        ws_plane_create_impacts) impacts_per_pitch of them, impact i at sub-bin
        i of the pitch; a single response with impacts_per_pitch > 1 is used
        for every impact (the degenerate case the reference pins)."""
        self.ctx, self.grid, self.response, self.n_sigma = ctx, grid, response, n_sigma
        self.lib = ctx.lib
        g = grid.to_c()
        h = C.c_void_p()
        if impacts_per_pitch == 1 and isinstance(response, ResponseParams):
            r, self._ww = response.to_c()
            check(self.lib.ws_plane_create(ctx.handle, C.byref(g), C.byref(r), n_sigma, C.byref(h)))
        else:
            rs = [response] * impacts_per_pitch if isinstance(response, ResponseParams) else list(response)
            if len(rs) != impacts_per_pitch:
                raise WsError(_lib.WS_EINVAL, "need one response per impact position")
            conv = [x.to_c() for x in rs]
            self._ww = [w for _, w in conv]
            arr = (_lib.ResponseC * len(rs))(*[c for c, _ in conv])
            check(self.lib.ws_plane_create_impacts(ctx.handle, C.byref(g), arr, impacts_per_pitch, n_sigma,
                                                   C.byref(h)))
        self.handle = h
        ctx._planes.add(self)
        info = _lib.PlaneInfoC()
        check(self.lib.ws_plane_get_info(h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in info._fields_}
        self.shape = (int(info.padded_wires), int(info.padded_ticks))

    def kernel(self) -> np.ndarray:
        k = np.zeros(int(self.info["n_lags"]), dtype=np.float64)
        check(self.lib.ws_plane_get_kernel(self.handle, k.ctypes.data, k.size))
        return k

    # ---- host-buffer entry points (synchronous)
    def simulate(self, depos, config: SimConfig, want_charge: bool = False, frame_out: np.ndarray | None = None):
        d = as_depos(depos)
        frame = frame_out if frame_out is not None else np.empty(self.shape, dtype=np.float32)
        charge = np.empty(self.shape, dtype=np.float32) if want_charge else None
        t = _lib.TimingC()
        opt = config.options()
        check(self.lib.ws_simulate_plane(self.handle, d.ctypes.data, len(d), C.byref(opt), frame.ctypes.data,
                                         charge.ctypes.data if charge is not None else None, C.byref(t)))
        return SimResult(frame=frame, charge=charge, timing=t.as_dict())

    def run(self, depos, config: SimConfig, adc_type: str = "i32", want_frame: bool = False,
            frame_type: str = "f32", want_charge: bool = False):
        """run_simulation (pipeline.cpp:345-427) on this plane: adc codes
        (int32 like SimResult::adc, or uint16), optionally the noisy frame
        before digitization and the charge grid (host buffers)."""
        d = as_depos(depos)
        r, _keep = config.readout(adc_type, frame_type)
        adc = np.empty(self.shape, dtype=np.uint16 if adc_type == "u16" else np.int32)
        frame = np.empty(self.shape, dtype=np.float64 if frame_type == "f64" else np.float32) if want_frame else None
        charge = np.empty(self.shape, dtype=np.float32) if want_charge else None
        t = _lib.TimingC()
        opt = config.options()
        check(self.lib.ws_run_simulation(self.handle, d.ctypes.data, len(d), C.byref(opt), C.byref(r),
                                         adc.ctypes.data, _ptr(frame), _ptr(charge), C.byref(t)))
        return RunResult(adc=adc, frame=frame, charge=charge, timing=t.as_dict(),
                         clipped_charge=int(t.clipped_charge))

    def run_device(self, depos_dev, n: int, config: SimConfig, adc_dev, frame_dev=None, charge_dev=None,
                   adc_type: str = "i32", frame_type: str = "f32", timing=None):
        r, _keep = config.readout(adc_type, frame_type)
        opt = config.options()
        check(self.lib.ws_run_simulation_device(self.handle, _ptr(depos_dev), n, C.byref(opt), C.byref(r),
                                                _ptr(adc_dev), _ptr(frame_dev), _ptr(charge_dev),
                                                C.byref(timing) if timing is not None else None))

    # ---- device entry points (torch tensors; asynchronous on the context stream)
    def simulate_device(self, depos_dev, n: int, config: SimConfig, frame_dev, charge_dev=None, timing=None,
                        charge_type: str = "f32"):
        opt = config.options(charge_type)
        check(self.lib.ws_simulate_plane_device(self.handle, _ptr(depos_dev), n, C.byref(opt), _ptr(frame_dev),
                                                _ptr(charge_dev), C.byref(timing) if timing is not None else None))

    def rasterize_device(self, depos_dev, n: int, config: SimConfig, charge_dev, timing=None):
        opt = config.options()
        check(self.lib.ws_rasterize_device(self.handle, _ptr(depos_dev), n, C.byref(opt), _ptr(charge_dev),
                                           C.byref(timing) if timing is not None else None))

    def convolve_device(self, charge_dev, frame_dev):
        check(self.lib.ws_convolve_device(self.handle, _ptr(charge_dev), _ptr(frame_dev)))

    def noise_digitize_device(self, frame_dev, sigma=0.0, seed=0, rng="substream", adc_dev=None, scale=1.0,
                              offset=2048.0, bits=12, spectrum=None):
        """add_noise (white with sigma, or spectrum mode with an amplitude
        spectrum; spectral.cpp:177-226) in place on a device frame, then
        digitize (spectral.cpp:228-238) into adc_dev (int32, nullable)."""
        amp = None
        if spectrum is not None:
            amp = np.ascontiguousarray(spectrum, dtype=np.float64)
            m = _lib.NoiseModelC(2, 1 if rng == "philox" else 0, 0.0, int(seed), amp.ctypes.data, amp.size)
        else:
            m = _lib.NoiseModelC(1 if sigma else 0, 1 if rng == "philox" else 0, float(sigma), int(seed), None, 0)
        check(self.lib.ws_noise_digitize_device(self.handle, _ptr(frame_dev), C.byref(m), scale, offset, bits,
                                                _ptr(adc_dev)))

    def close(self):
        if self.handle:
            self.lib.ws_plane_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return C.c_void_p(x)
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        return C.c_void_p(x.ctypes.data)
    raise TypeError(f"cannot take a pointer of {type(x)}")


@dataclass
class SimResult:
    frame: np.ndarray            # pre-noise measurement M (float32, padded)
    charge: np.ndarray | None    # charge grid S (float32, padded)
    timing: dict


@dataclass
class RunResult:
    """SimResult (pipeline.hpp:94-99): adc codes, the charge grid (optional),
    clipped charge; plus the noisy frame before digitization (optional)."""
    adc: np.ndarray
    frame: np.ndarray | None
    charge: np.ndarray | None
    timing: dict
    clipped_charge: int


def simulate_event(ctx: Context, planes: Sequence[Plane], depos: Sequence, config: SimConfig,
                   frames: Sequence[np.ndarray] | None = None):
    """Independent planes of one event through one batch of launches (host buffers)."""
    n = len(planes)
    ds = [as_depos(d) for d in depos]
    frames = list(frames) if frames is not None else [np.empty(p.shape, dtype=np.float32) for p in planes]
    PArr = C.c_void_p * n
    parr = PArr(*[p.handle.value for p in planes])
    darr = PArr(*[d.ctypes.data for d in ds])
    narr = (C.c_uint64 * n)(*[len(d) for d in ds])
    farr = PArr(*[f.ctypes.data for f in frames])
    t = _lib.TimingC()
    opt = config.options()
    check(ctx.lib.ws_simulate_event(ctx.handle, n, parr, darr, narr, C.byref(opt), farr, C.byref(t)))
    return frames, t.as_dict()


def simulate_events(ctx: Context, planes: Sequence[Plane], events: Sequence[Sequence], config: SimConfig,
                    frames: Sequence[Sequence[np.ndarray]] | None = None):
    """A batch of events (each a per-plane list of depo arrays) through the
    pipelined host-buffer path (ws_simulate_events). Returns frames[e][p]."""
    n_ev, n_pl = len(events), len(planes)
    ds = [as_depos(d) for ev in events for d in ev]
    if frames is None:
        frames = [[np.empty(p.shape, dtype=np.float32) for p in planes] for _ in range(n_ev)]
    flat = [f for ev in frames for f in ev]
    PArr = C.c_void_p * n_pl
    parr = PArr(*[p.handle.value for p in planes])
    DArr = C.c_void_p * (n_ev * n_pl)
    darr = DArr(*[d.ctypes.data for d in ds])
    narr = (C.c_uint64 * (n_ev * n_pl))(*[len(d) for d in ds])
    farr = DArr(*[f.ctypes.data for f in flat])
    t = _lib.TimingC()
    opt = config.options()
    check(ctx.lib.ws_simulate_events(ctx.handle, n_ev, n_pl, parr, darr, narr, C.byref(opt), farr, C.byref(t)))
    return frames, t.as_dict()


def run_events(ctx: Context, planes: Sequence[Plane], events: Sequence[Sequence], config: SimConfig,
               adc_type: str = "i32", want_frame: bool = False, frame_type: str = "f32", adcs=None, frames=None):
    """run_simulation over a batch of events (ws_run_events, pipelined host
    buffers): returns (adcs[e][p], frames[e][p] or None, timing)."""
    n_ev, n_pl = len(events), len(planes)
    ds = [as_depos(d) for ev in events for d in ev]
    adt = np.uint16 if adc_type == "u16" else np.int32
    if adcs is None:
        adcs = [[np.empty(p.shape, dtype=adt) for p in planes] for _ in range(n_ev)]
    if frames is None and want_frame:
        fdt = np.float64 if frame_type == "f64" else np.float32
        frames = [[np.empty(p.shape, dtype=fdt) for p in planes] for _ in range(n_ev)]
    PArr = C.c_void_p * n_pl
    parr = PArr(*[p.handle.value for p in planes])
    DArr = C.c_void_p * (n_ev * n_pl)
    darr = DArr(*[d.ctypes.data for d in ds])
    narr = (C.c_uint64 * (n_ev * n_pl))(*[len(d) for d in ds])
    aarr = DArr(*[a.ctypes.data for ev in adcs for a in ev])
    farr = DArr(*[f.ctypes.data for ev in frames for f in ev]) if frames is not None else None
    r, _keep = config.readout(adc_type, frame_type)
    t = _lib.TimingC()
    opt = config.options()
    check(ctx.lib.ws_run_events(ctx.handle, n_ev, n_pl, parr, darr, narr, C.byref(opt), C.byref(r), aarr, farr,
                                C.byref(t)))
    return adcs, frames, t.as_dict()


class Multi:
    """Several GPUs of one node (ws_multi_*): a context per device (a device
    may repeat), the same plane specs on each, a host thread per device;
    independent events or (face, plane) units sharded by LPT, outputs
    gathered into the caller's host buffers. No data crosses devices."""

    def __init__(self, devices: Sequence[int], specs: Sequence[tuple], n_sigma: float = 3.0):
        self.lib = _lib.load()
        self.specs = list(specs)
        g = (_lib.GridSpecC * len(specs))(*[gs.to_c() for gs, _ in specs])
        rs = [r.to_c() for _, r in specs]
        self._ww = [w for _, w in rs]
        r = (_lib.ResponseC * len(specs))(*[rc for rc, _ in rs])
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        check(self.lib.ws_multi_create(len(devices), devs, len(specs), g, r, n_sigma, C.byref(h)))
        self.handle = h
        self.n_devices = len(devices)
        self.shapes = [(gs.padded_wires(), gs.padded_ticks()) for gs, _ in specs]

    def set_conv_path(self, path: str):
        check(self.lib.ws_multi_set_conv_path(self.handle, Context.CONV_PATHS[path]))

    def run_events(self, events: Sequence[Sequence], config: SimConfig, adc_type: str | None = None):
        """events[e][p] depo arrays. adc_type None: fp32 frames; else ADC codes
        ("i32" / "u16"). Returns (outputs[e][p], device index per event)."""
        n_ev, n_pl = len(events), len(self.specs)
        ds = [as_depos(d) for ev in events for d in ev]
        if adc_type is None:
            outs = [[np.empty(sh, dtype=np.float32) for sh in self.shapes] for _ in range(n_ev)]
        else:
            dt = np.uint16 if adc_type == "u16" else np.int32
            outs = [[np.empty(sh, dtype=dt) for sh in self.shapes] for _ in range(n_ev)]
        A = C.c_void_p * (n_ev * n_pl)
        darr = A(*[d.ctypes.data for d in ds])
        narr = (C.c_uint64 * (n_ev * n_pl))(*[len(d) for d in ds])
        oarr = A(*[o.ctypes.data for ev in outs for o in ev])
        where = (C.c_uint32 * n_ev)()
        opt = config.options()
        if adc_type is None:
            check(self.lib.ws_multi_run_events(self.handle, n_ev, darr, narr, C.byref(opt), None, None, oarr, where,
                                               None))
        else:
            r, _keep = config.readout(adc_type)
            check(self.lib.ws_multi_run_events(self.handle, n_ev, darr, narr, C.byref(opt), C.byref(r), oarr, None,
                                               where, None))
        return outs, list(where)

    def run_units(self, plane_of: Sequence[int], depos: Sequence, config: SimConfig):
        """Independent plane runs (unit u on plane spec plane_of[u]), fp32
        frames. Returns (frames[u], device index per unit)."""
        n = len(plane_of)
        ds = [as_depos(d) for d in depos]
        outs = [np.empty(self.shapes[p], dtype=np.float32) for p in plane_of]
        A = C.c_void_p * n
        where = (C.c_uint32 * n)()
        opt = config.options()
        check(self.lib.ws_multi_run_units(self.handle, n, (C.c_uint32 * n)(*plane_of), A(*[d.ctypes.data for d in ds]),
                                          (C.c_uint64 * n)(*[len(d) for d in ds]), C.byref(opt), None, None,
                                          A(*[o.ctypes.data for o in outs]), where))
        return outs, list(where)

    def close(self):
        if self.handle:
            self.lib.ws_multi_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def simulate_event_device(ctx: Context, planes: Sequence[Plane], depos_dev: Sequence, n_depos: Sequence[int],
                          config: SimConfig, frames_dev: Sequence, timing=None):
    n = len(planes)
    PArr = C.c_void_p * n
    parr = PArr(*[p.handle.value for p in planes])
    darr = PArr(*[_ptr(d).value for d in depos_dev])
    narr = (C.c_uint64 * n)(*n_depos)
    farr = PArr(*[_ptr(f).value for f in frames_dev])
    opt = config.options()
    check(ctx.lib.ws_simulate_event_device(ctx.handle, n, parr, darr, narr, C.byref(opt), farr,
                                           C.byref(timing) if timing is not None else None))


def run_simulation(config: SimConfig, depos, device: int = 0, ctx: Context | None = None,
                   adc_type: str = "i32", want_frame: bool = False) -> RunResult:
    """run_simulation (pipeline.hpp:104) on the GPU: SimResult's adc,
    charge grid and clipped charge (+ the noisy frame if asked)."""
    ctx = ctx or Context(device)
    plane = Plane(ctx, config.grid, config.response, config.n_sigma)
    try:
        return plane.run(depos, config, adc_type=adc_type, want_frame=want_frame, want_charge=True)
    finally:
        plane.close()


def gen_depos(n: int, seed: int, grid: GridSpec, ranges: Sequence[float] | None = None) -> np.ndarray:
    """The reference's gen_depos (pipeline.cpp:264-294), same xoshiro stream."""
    lib = _lib.load()
    out = np.zeros(n, dtype=DEPO_DTYPE)
    g = grid.to_c()
    r = None if ranges is None else np.ascontiguousarray(ranges, dtype=np.float64)
    check(lib.ws_gen_depos_uniform(n, seed, C.byref(g), r.ctypes.data if r is not None else None, out.ctypes.data))
    return out


def load_depos(path) -> np.ndarray:
    """load_depos (pipeline.cpp:226-262) through the native CSV reader: same
    format and validation; a bad file raises WsError (WS_ERUNTIME)."""
    lib = _lib.load()
    ptr = C.c_void_p()
    n = C.c_uint64()
    check(lib.ws_load_depos_csv(str(path).encode(), 0, C.byref(ptr), C.byref(n)))
    try:
        out = np.empty(n.value, dtype=DEPO_DTYPE)
        if n.value:
            C.memmove(out.ctypes.data, ptr.value, n.value * DEPO_DTYPE.itemsize)
        return out
    finally:
        lib.ws_free_depos(ptr, 0)


def save_depos(path, depos) -> None:
    """gen_depos's CSV writer (pipeline.cpp:270-293), %.17g fields."""
    lib = _lib.load()
    d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
    check(lib.ws_save_depos_csv(str(path).encode(), d.ctypes.data if len(d) else None, len(d)))


# ---- signal processing (sigproc.hpp; the paper's Listing 1) ----------------

@dataclass
class ChainResult:
    """ChainResult (sigproc.hpp:53-57)."""
    block: np.ndarray
    medians: np.ndarray
    max_rel_imag: float


def sigproc_chain(data, filt, pad_rows: int = 0, out_rows: int | None = None, ctx: Context | None = None,
                  want_medians: bool = True, block_out: np.ndarray | None = None,
                  medians_out: np.ndarray | None = None) -> ChainResult:
    """sigproc_chain (sigproc.cpp:104-118) on the GPU through host buffers:
    filter -> inverse DFT along rows (real part) -> rows [pad_rows, pad_rows +
    out_rows) -> per-row medians. data: (rows, cols) complex128; filt: cols
    real or complex values."""
    ctx = ctx or Context()
    data = np.ascontiguousarray(data, dtype=np.complex128)
    if data.ndim != 2:
        raise WsError(_lib.WS_EINVAL, "SignalBatch: data must be 2-D")
    rows, cols = data.shape
    out_rows = rows - pad_rows if out_rows is None else out_rows
    f = np.asarray(filt)
    is_complex = np.iscomplexobj(f)
    f = np.ascontiguousarray(f, dtype=np.complex128 if is_complex else np.float64).reshape(-1)
    block = np.empty((max(out_rows, 0), cols), dtype=np.float64) if block_out is None else block_out
    if block.shape != (max(out_rows, 0), cols) or block.dtype != np.float64 or not block.flags.c_contiguous:
        raise WsError(_lib.WS_EINVAL, "block_out must be a C-contiguous float64 (out_rows, cols) array")
    med = None
    if want_medians:
        med = np.empty(max(out_rows, 0), dtype=np.float64) if medians_out is None else medians_out
    mri = C.c_double()
    b = _lib.SignalBatchC(data.ctypes.data, rows, cols, pad_rows, out_rows)
    check(ctx.lib.ws_sigproc_chain(ctx.handle, C.byref(b), f.ctypes.data, f.size, int(is_complex),
                                   block.ctypes.data, med.ctypes.data if med is not None else None, C.byref(mri)))
    return ChainResult(block, med, mri.value)


def sigproc_chain_device(ctx: Context, data_dev, rows: int, cols: int, filter_dev, block_dev, medians_dev=None,
                         pad_rows: int = 0, out_rows: int | None = None, residue: bool = False):
    """Device-pointer form (asynchronous unless residue=True, which returns
    max_rel_imag). data_dev: rows x cols complex128; filter_dev: cols complex128."""
    out_rows = rows - pad_rows if out_rows is None else out_rows
    b = _lib.SignalBatchC(_ptr(data_dev).value, rows, cols, pad_rows, out_rows)
    mri = C.c_double()
    check(ctx.lib.ws_sigproc_chain_device(ctx.handle, C.byref(b), _ptr(filter_dev), cols, _ptr(block_dev),
                                          _ptr(medians_dev), C.byref(mri) if residue else None))
    return mri.value if residue else None


def row_medians_device(ctx: Context, m_dev, rows: int, cols: int, medians_dev):
    """row_median (sigproc.cpp:80-93) of every row of a real rows x cols device matrix."""
    check(ctx.lib.ws_row_medians_device(ctx.handle, _ptr(m_dev), rows, cols, _ptr(medians_dev)))


def sigproc_max_cols() -> int:
    return int(_lib.load().ws_sigproc_max_cols())
