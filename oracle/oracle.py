"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes bindings for the two CPU checkers of the hot path:

* ``Oracle``   -> oracle/liboracle.so, the plain-C restatement (wsoracle.c), built
  from committed source on any box (gcc is in the image);
* ``Reference`` -> oracle/_ref/libwsref.so, the UNMODIFIED reference library
  (/root/reference/proj/src) + ref_harness.cpp, built here by ``make ref``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline / reference
arm may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libwsref.so"

DEPO_DTYPE = np.dtype(
    [("id", "<i8"), ("t", "<f8"), ("x", "<f8"), ("q", "<i8"), ("sigma_t", "<f8"), ("sigma_x", "<f8")]
)


class Grid(C.Structure):
    _fields_ = [
        ("n_wires", C.c_uint64), ("n_ticks", C.c_uint64), ("pad_wires", C.c_uint64), ("pad_ticks", C.c_uint64),
        ("pitch", C.c_double), ("tick", C.c_double), ("origin_x", C.c_double), ("origin_t", C.c_double),
    ]


class Response(C.Structure):
    _fields_ = [
        ("plane_kind", C.c_int32), ("shaper_order", C.c_int32), ("field_sigma_t", C.c_double),
        ("shaper_peaking", C.c_double), ("gain", C.c_double), ("wire_weights", C.POINTER(C.c_double)),
        ("n_wire_weights", C.c_uint64),
    ]


class Drift(C.Structure):
    _fields_ = [("response_plane_x", C.c_double), ("drift_speed", C.c_double),
                ("diffusion_long", C.c_double), ("diffusion_tran", C.c_double)]


def make_grid(n_wires=1000, n_ticks=6000, pad_wires=100, pad_ticks=100, pitch=5.0, tick=0.5, origin_x=0.0,
              origin_t=0.0) -> Grid:
    return Grid(n_wires, n_ticks, pad_wires, pad_ticks, pitch, tick, origin_x, origin_t)


def make_response(plane_kind="collection", field_sigma_t=1.0, shaper_peaking=2.0, shaper_order=2, gain=14.0,
                  wire_weights=(1.0,)) -> Response:
    ww = np.ascontiguousarray(np.asarray(wire_weights, dtype=np.float64))
    r = Response(1 if plane_kind == "collection" else 0, shaper_order, field_sigma_t, shaper_peaking, gain,
                 ww.ctypes.data_as(C.POINTER(C.c_double)), ww.size)
    r._keep = ww  # keep the weights alive with the struct
    return r


def padded(g: Grid):
    return int(g.n_wires + 2 * g.pad_wires), int(g.n_ticks + 2 * g.pad_ticks)


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def fnv1a64(a: np.ndarray) -> int:
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(a).view(np.uint8).tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def build_oracle(force: bool = False) -> Path:
    if force or not ORACLE_SO.exists() or ORACLE_SO.stat().st_mtime < (HERE / "wsoracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "liboracle.so"], check=True, capture_output=True)
    return ORACLE_SO


class OracleError(RuntimeError):
    pass


class Oracle:
    """The C restatement (wsoracle.c)."""

    def __init__(self):
        self.lib = C.CDLL(str(build_oracle()))
        L = self.lib
        L.wso_last_error.restype = C.c_char_p
        L.wso_fnv1a64.restype = C.c_uint64
        L.wso_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        L.wso_uniform01.restype = C.c_double
        L.wso_src_uniform.restype = C.c_double
        L.wso_src_normal.restype = C.c_double
        L.wso_src_init.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64]
        L.wso_src_uniform.argtypes = [C.c_void_p]
        L.wso_src_normal.argtypes = [C.c_void_p]
        L.wso_binomial.argtypes = [C.c_int64, C.c_double, C.c_void_p, C.POINTER(C.c_int64)]
        L.wso_sample_patch.argtypes = [C.POINTER(Grid), C.c_void_p, C.c_double, C.c_void_p, C.c_void_p,
                                       C.c_size_t, C.POINTER(C.c_double)]
        L.wso_map_depo.argtypes = [C.POINTER(Grid), C.c_void_p, C.c_double, C.c_void_p]
        L.wso_drift_depo.argtypes = [C.c_void_p, C.POINTER(Drift), C.c_void_p]
        L.wso_charge_fluct_off.argtypes = [C.POINTER(Grid), C.c_void_p, C.c_size_t, C.c_double, C.POINTER(Drift),
                                           C.c_void_p, C.POINTER(C.c_int64)]
        L.wso_charge_fluct_on.argtypes = [C.POINTER(Grid), C.c_void_p, C.c_size_t, C.c_double, C.POINTER(Drift),
                                          C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.POINTER(C.c_int64)]
        L.wso_response_td.argtypes = [C.POINTER(Grid), C.POINTER(Response), C.c_void_p, C.c_size_t,
                                      C.POINTER(C.c_long), C.POINTER(C.c_size_t), C.POINTER(C.c_long),
                                      C.POINTER(C.c_long)]
        L.wso_convolve_direct.argtypes = [C.POINTER(Grid), C.POINTER(Response), C.c_void_p, C.c_void_p]
        L.wso_add_white_noise.argtypes = [C.POINTER(Grid), C.c_double, C.c_uint64, C.c_void_p]
        L.wso_add_white_noise_rng.argtypes = [C.POINTER(Grid), C.c_double, C.c_uint64, C.c_int, C.c_void_p]
        L.wso_digitize.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.c_double, C.c_int, C.c_void_p]
        L.wso_philox4x32_10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.wso_sigproc_chain.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
        L.wso_row_median.restype = C.c_double
        L.wso_row_median.argtypes = [C.c_void_p, C.c_size_t]

    def _check(self, rc):
        if rc:
            raise OracleError(self.lib.wso_last_error().decode())

    # --- rng
    def philox(self, ctr, key):
        c = np.asarray(ctr, dtype=np.uint32)
        k = np.asarray(key, dtype=np.uint32)
        o = np.zeros(4, dtype=np.uint32)
        self.lib.wso_philox4x32_10(_p(c), _p(k), _p(o))
        return o

    def draws(self, mode, kind, seed, stream_id, count):
        src = (C.c_char * 128)()
        self.lib.wso_src_init(src, mode, seed, stream_id)
        f = self.lib.wso_src_normal if kind else self.lib.wso_src_uniform
        return np.array([f(src) for _ in range(count)])

    def binomials(self, n, p, seed, stream_id, count, mode=0):
        src = (C.c_char * 128)()
        self.lib.wso_src_init(src, mode, seed, stream_id)
        out = np.zeros(count, dtype=np.int64)
        k = C.c_int64()
        for i in range(count):
            self._check(self.lib.wso_binomial(n, p, src, C.byref(k)))
            out[i] = k.value
        return out

    # --- rasterize
    def map_depo(self, g, depo, n_sigma=3.0):
        d = np.asarray([depo], dtype=DEPO_DTYPE) if not isinstance(depo, np.ndarray) else depo.reshape(1)
        out = np.zeros(6, dtype=np.int64)
        self._check(self.lib.wso_map_depo(C.byref(g), _p(d), n_sigma, _p(out)))
        return out

    def drift(self, depos, drift: Drift):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        out = d.copy()
        for i in range(len(d)):
            self._check(self.lib.wso_drift_depo(C.c_void_p(d.ctypes.data + 48 * i), C.byref(drift),
                                                C.c_void_p(out.ctypes.data + 48 * i)))
        return out

    def sample_patch(self, g, depo, n_sigma=3.0, cap=1 << 16):
        d = np.ascontiguousarray(np.asarray(depo, dtype=DEPO_DTYPE).reshape(1))
        meta = np.zeros(5, dtype=np.int64)
        vals = np.zeros(cap, dtype=np.float64)
        captured = C.c_double()
        self._check(self.lib.wso_sample_patch(C.byref(g), _p(d), n_sigma, _p(meta), _p(vals), cap,
                                              C.byref(captured)))
        nw, nt = int(meta[2]), int(meta[3])
        return dict(wire_offset=int(meta[0]), tick_offset=int(meta[1]), n_w=nw, n_t=nt, clipped=bool(meta[4]),
                    values=vals[: nw * nt].reshape(nw, nt).copy(), captured_mass=captured.value)

    def charge_fluct_off(self, g, depos, n_sigma=3.0, drift: Drift | None = None):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        W, T = padded(g)
        s = np.zeros((W, T), dtype=np.float64)
        clipped = C.c_int64()
        self._check(self.lib.wso_charge_fluct_off(C.byref(g), _p(d), len(d), n_sigma,
                                                  C.byref(drift) if drift else None, _p(s), C.byref(clipped)))
        return s, clipped.value

    def charge_fluct_on(self, g, depos, n_sigma=3.0, rng_mode=0, approx=False, seed=12345,
                        drift: Drift | None = None):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        W, T = padded(g)
        s = np.zeros((W, T), dtype=np.int64)
        clipped = C.c_int64()
        self._check(self.lib.wso_charge_fluct_on(C.byref(g), _p(d), len(d), n_sigma,
                                                 C.byref(drift) if drift else None, rng_mode, int(approx), seed,
                                                 _p(s), C.byref(clipped)))
        return s, clipped.value

    # --- response / convolve
    def response_td(self, g, r):
        lo, nl, st, sw = C.c_long(), C.c_size_t(), C.c_long(), C.c_long()
        self._check(self.lib.wso_response_td(C.byref(g), C.byref(r), None, 0, C.byref(lo), C.byref(nl),
                                             C.byref(st), C.byref(sw)))
        k = np.zeros(nl.value, dtype=np.float64)
        self._check(self.lib.wso_response_td(C.byref(g), C.byref(r), _p(k), k.size, C.byref(lo), C.byref(nl),
                                             C.byref(st), C.byref(sw)))
        return dict(kernel=k, lo_lag=lo.value, support_ticks=st.value, support_wires=sw.value)

    def convolve(self, g, r, s):
        s = np.ascontiguousarray(s, dtype=np.float64)
        m = np.zeros_like(s)
        self._check(self.lib.wso_convolve_direct(C.byref(g), C.byref(r), _p(s), _p(m)))
        return m

    def sigproc_chain(self, data, filt, pad_rows, out_rows, medians=True):
        """sigproc_chain restated (sigproc.cpp:104-118): (block, medians, max_rel_imag)."""
        data = np.ascontiguousarray(data, dtype=np.complex128)
        filt = np.ascontiguousarray(np.broadcast_to(filt, (data.shape[1],)), dtype=np.complex128)
        rows, cols = data.shape
        block = np.zeros((out_rows, cols))
        med = np.zeros(out_rows) if medians else None
        mri = C.c_double()
        self._check(self.lib.wso_sigproc_chain(_p(data), rows, cols, pad_rows, out_rows, _p(filt), _p(block),
                                               _p(med) if medians else None, C.byref(mri)))
        return block, med, mri.value

    def row_median(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return self.lib.wso_row_median(_p(v), v.size)

    def add_white_noise(self, g, m, sigma, seed, rng_mode=0):
        out = np.ascontiguousarray(m, dtype=np.float64).copy()
        self._check(self.lib.wso_add_white_noise_rng(C.byref(g), sigma, seed, rng_mode, _p(out)))
        return out

    def digitize(self, m, scale=1.0, offset=2048.0, bits=12):
        m = np.ascontiguousarray(m, dtype=np.float64)
        adc = np.zeros(m.shape, dtype=np.int32)
        self._check(self.lib.wso_digitize(_p(m), m.size, scale, offset, bits, _p(adc)))
        return adc


def ref_available() -> bool:
    return REF_SO.exists()


def build_ref() -> Path | None:
    """Compile the unmodified reference into oracle/_ref (only where /root/reference exists)."""
    ref_src = Path(os.environ.get("WS_REFERENCE", "/root/reference")) / "proj"
    if not ref_src.exists():
        return REF_SO if REF_SO.exists() else None
    subprocess.run(["make", "-C", str(HERE), "ref", f"REF={ref_src}", "-j8"], check=True, capture_output=True)
    # the drop-in check program (reference types -> B200 library and reference), once libwsgpu.so exists
    if (HERE.parent / "paper_2104_08265_b200" / "libwsgpu.so").exists():
        r = subprocess.run(["make", "-C", str(HERE), "dropin", f"REF={ref_src}"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("make dropin failed:\n" + r.stdout + r.stderr)
    return REF_SO


class Reference:
    """The unmodified reference library through ref_harness.cpp."""

    def __init__(self):
        if not REF_SO.exists():
            raise OracleError(f"{REF_SO} not built (make -C oracle ref)")
        self.lib = C.CDLL(str(REF_SO))
        L = self.lib
        L.wsr_last_error.restype = C.c_char_p
        G, R = C.POINTER(Grid), C.POINTER(Response)
        L.wsr_run_simulation.argtypes = [G, R, C.c_void_p, C.c_uint64, C.c_double, C.c_int, C.c_uint64,
                                         C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                         C.c_double, C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_int,
                                         C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p]
        L.wsr_sample_patch.argtypes = [G, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_uint64,
                                       C.POINTER(C.c_double)]
        L.wsr_map_depo.argtypes = [G, C.c_void_p, C.c_double, C.c_void_p]
        L.wsr_drift.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.wsr_build_response.argtypes = [G, R, C.c_void_p, C.c_void_p]
        L.wsr_convolve_int.argtypes = [G, R, C.c_void_p, C.c_void_p, C.c_int]
        L.wsr_convolve_real.argtypes = [G, R, C.c_void_p, C.c_void_p, C.c_int]
        L.wsr_fluct_off_charge.argtypes = [G, C.c_void_p, C.c_uint64, C.c_double, C.c_int, C.c_void_p, C.c_void_p,
                                           C.POINTER(C.c_int64)]
        L.wsr_fluct_philox_charge.argtypes = [G, C.c_void_p, C.c_uint64, C.c_double, C.c_uint64, C.c_int,
                                              C.c_void_p, C.POINTER(C.c_int64)]
        L.wsr_gen_depos.argtypes = [C.c_uint64, C.c_uint64, G, C.c_void_p]
        L.wsr_gen_depos_csv.argtypes = [C.c_uint64, C.c_uint64, G, C.c_char_p]
        L.wsr_load_depos.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.wsr_sigproc_chain.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p,
                                        C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
        L.wsr_row_median.restype = C.c_double
        L.wsr_row_median.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
        L.wsr_draws.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
        L.wsr_binomials.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
        L.wsr_philox4x32_10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.wsr_noise_digitize.argtypes = [G, C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_uint64, C.c_uint64,
                                         C.c_double, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.wsr_time_fluct_off.argtypes = [G, R, C.c_void_p, C.c_uint64, C.c_double, C.c_int, C.c_void_p,
                                         C.c_void_p]
        L.wsr_plane_create.restype = C.c_void_p
        L.wsr_plane_create.argtypes = [G, R, C.POINTER(C.c_double)]
        L.wsr_plane_destroy.argtypes = [C.c_void_p]
        L.wsr_plane_time_fluct_off.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_int, C.c_void_p,
                                               C.c_void_p]

    def _check(self, rc):
        if rc:
            raise OracleError(self.lib.wsr_last_error().decode())

    def gen_depos(self, n, seed, g):
        out = np.zeros(n, dtype=DEPO_DTYPE)
        self._check(self.lib.wsr_gen_depos(n, seed, C.byref(g), _p(out)))
        return out

    def sigproc_chain(self, data, filt, pad_rows, out_rows, workers=1):
        """sigproc_chain (sigproc.cpp:104-118): (block, medians, max_rel_imag, seconds)."""
        data = np.ascontiguousarray(data, dtype=np.complex128)
        filt = np.ascontiguousarray(np.broadcast_to(filt, (data.shape[1],)), dtype=np.complex128)
        rows, cols = data.shape
        block = np.zeros((out_rows, cols))
        med = np.zeros(out_rows)
        mri, sec = C.c_double(), C.c_double()
        self._check(self.lib.wsr_sigproc_chain(_p(data), rows, cols, pad_rows, out_rows, _p(filt), workers,
                                               _p(block), _p(med), C.byref(mri), C.byref(sec)))
        return block, med, mri.value, sec.value

    def row_median(self, v, by_sort=False):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return self.lib.wsr_row_median(_p(v), v.size, int(by_sort))

    def gen_depos_csv(self, n, seed, g, path):
        self._check(self.lib.wsr_gen_depos_csv(n, seed, C.byref(g), str(path).encode()))

    def load_depos(self, path, cap=1 << 20):
        out = np.zeros(cap, dtype=DEPO_DTYPE)
        n = C.c_uint64()
        self._check(self.lib.wsr_load_depos(str(path).encode(), _p(out), cap, C.byref(n)))
        return out[:n.value].copy()

    def draws(self, mode, kind, seed, stream_id, count):
        out = np.zeros(count, dtype=np.float64)
        self._check(self.lib.wsr_draws(mode, kind, seed, stream_id, count, _p(out)))
        return out

    def binomials(self, n, p, seed, stream_id, count):
        out = np.zeros(count, dtype=np.int64)
        self._check(self.lib.wsr_binomials(n, p, seed, stream_id, count, _p(out)))
        return out

    def philox(self, ctr, key):
        c = np.asarray(ctr, dtype=np.uint32)
        k = np.asarray(key, dtype=np.uint32)
        o = np.zeros(4, dtype=np.uint32)
        self.lib.wsr_philox4x32_10(_p(c), _p(k), _p(o))
        return o

    def sample_patch(self, g, depo, n_sigma=3.0, cap=1 << 16):
        d = np.ascontiguousarray(np.asarray(depo, dtype=DEPO_DTYPE).reshape(1))
        meta = np.zeros(5, dtype=np.int64)
        vals = np.zeros(cap, dtype=np.float64)
        captured = C.c_double()
        self._check(self.lib.wsr_sample_patch(C.byref(g), _p(d), n_sigma, _p(meta), _p(vals), cap,
                                              C.byref(captured)))
        nw, nt = int(meta[2]), int(meta[3])
        return dict(wire_offset=int(meta[0]), tick_offset=int(meta[1]), n_w=nw, n_t=nt, clipped=bool(meta[4]),
                    values=vals[: nw * nt].reshape(nw, nt).copy(), captured_mass=captured.value)

    def map_depo(self, g, depo, n_sigma=3.0):
        d = np.ascontiguousarray(np.asarray(depo, dtype=DEPO_DTYPE).reshape(1))
        out = np.zeros(6, dtype=np.int64)
        self._check(self.lib.wsr_map_depo(C.byref(g), _p(d), n_sigma, _p(out)))
        return out

    def drift(self, depos, drift: Drift):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        out = d.copy()
        p = np.array([drift.response_plane_x, drift.drift_speed, drift.diffusion_long, drift.diffusion_tran])
        for i in range(len(d)):
            self._check(self.lib.wsr_drift(C.c_void_p(d.ctypes.data + 48 * i), _p(p),
                                           C.c_void_p(out.ctypes.data + 48 * i)))
        return out

    def run_simulation(self, g, r, depos, n_sigma=3.0, rng_mode=2, seed=12345, slice_len=1024, dispatch=0,
                       workers=1, scatter_atomic=0, drift: Drift | None = None, noise_mode=0, noise_sigma=0.0,
                       noise_spectrum=None, adc=(1.0, 2048.0, 12)):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        W, T = padded(g)
        charge = np.zeros((W, T), dtype=np.int64)
        adc_out = np.zeros((W, T), dtype=np.int32)
        clipped = C.c_int64()
        timing = np.zeros(6, dtype=np.float64)
        dp = (np.array([drift.response_plane_x, drift.drift_speed, drift.diffusion_long, drift.diffusion_tran])
              if drift else np.zeros(4))
        spec = None if noise_spectrum is None else np.ascontiguousarray(noise_spectrum, dtype=np.float64)
        self._check(self.lib.wsr_run_simulation(
            C.byref(g), C.byref(r), _p(d), len(d), n_sigma, rng_mode, seed, slice_len, dispatch, workers,
            scatter_atomic, 1 if drift else 0, _p(dp), noise_mode, noise_sigma, _p(spec),
            0 if spec is None else spec.size, adc[0], adc[1], adc[2], _p(charge), _p(adc_out), C.byref(clipped),
            _p(timing)))
        return dict(charge=charge, adc=adc_out, clipped_charge=clipped.value, timing=timing)

    def build_response(self, g, r, values=True):
        W, T = padded(g)
        vals = np.zeros((W, T), dtype=np.complex128) if values else None
        sup = np.zeros(2, dtype=np.int64)
        self._check(self.lib.wsr_build_response(C.byref(g), C.byref(r), _p(vals), _p(sup)))
        return dict(values=vals, support_ticks=int(sup[0]), support_wires=int(sup[1]))

    def convolve_int(self, g, r, s, workers=1):
        s = np.ascontiguousarray(s, dtype=np.int64)
        m = np.zeros(s.shape, dtype=np.float64)
        self._check(self.lib.wsr_convolve_int(C.byref(g), C.byref(r), _p(s), _p(m), workers))
        return m

    def convolve_real(self, g, r, s, workers=1):
        s = np.ascontiguousarray(s, dtype=np.float64)
        m = np.zeros(s.shape, dtype=np.float64)
        self._check(self.lib.wsr_convolve_real(C.byref(g), C.byref(r), _p(s), _p(m), workers))
        return m

    def charge_fluct_off(self, g, depos, n_sigma=3.0, drift: Drift | None = None):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        W, T = padded(g)
        s = np.zeros((W, T), dtype=np.float64)
        clipped = C.c_int64()
        dp = (np.array([drift.response_plane_x, drift.drift_speed, drift.diffusion_long, drift.diffusion_tran])
              if drift else np.zeros(4))
        self._check(self.lib.wsr_fluct_off_charge(C.byref(g), _p(d), len(d), n_sigma, 1 if drift else 0, _p(dp),
                                                  _p(s), C.byref(clipped)))
        return s, clipped.value

    def charge_fluct_philox(self, g, depos, n_sigma=3.0, seed=12345, approx=False):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        W, T = padded(g)
        s = np.zeros((W, T), dtype=np.int64)
        clipped = C.c_int64()
        self._check(self.lib.wsr_fluct_philox_charge(C.byref(g), _p(d), len(d), n_sigma, seed, int(approx), _p(s),
                                                     C.byref(clipped)))
        return s, clipped.value

    def noise_digitize(self, g, m, noise_mode=1, sigma=0.0, spectrum=None, seed=12345, adc=(1.0, 2048.0, 12),
                       workers=1):
        m = np.ascontiguousarray(m, dtype=np.float64)
        noisy = np.zeros_like(m)
        a = np.zeros(m.shape, dtype=np.int32)
        spec = None if spectrum is None else np.ascontiguousarray(spectrum, dtype=np.float64)
        self._check(self.lib.wsr_noise_digitize(C.byref(g), _p(m), noise_mode, sigma, _p(spec),
                                                0 if spec is None else spec.size, seed, adc[0], adc[1], adc[2],
                                                _p(noisy), _p(a), workers))
        return noisy, a

    def plane(self, g, r):
        """Cached response kernel for repeated timing (RefPlane)."""
        b = C.c_double()
        h = self.lib.wsr_plane_create(C.byref(g), C.byref(r), C.byref(b))
        if not h:
            raise OracleError(self.lib.wsr_last_error().decode())
        return RefPlane(self, h, padded(g), b.value)

    def time_fluct_off(self, g, r, depos, n_sigma=3.0, workers=1, want_m=False):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        W, T = padded(g)
        m = np.zeros((W, T), dtype=np.float64) if want_m else None
        times = np.zeros(4, dtype=np.float64)
        self._check(self.lib.wsr_time_fluct_off(C.byref(g), C.byref(r), _p(d), len(d), n_sigma, workers, _p(m),
                                                _p(times)))
        return dict(sample_s=times[0], scatter_s=times[1], convolve_s=times[2], build_response_s=times[3], m=m)


class RefPlane:
    def __init__(self, ref, handle, shape, build_s):
        self.ref, self.handle, self.shape, self.build_s = ref, handle, shape, build_s

    def time_fluct_off(self, depos, n_sigma=3.0, workers=1, want_m=False):
        d = np.ascontiguousarray(depos, dtype=DEPO_DTYPE)
        m = np.zeros(self.shape, dtype=np.float64) if want_m else None
        times = np.zeros(3, dtype=np.float64)
        self.ref._check(self.ref.lib.wsr_plane_time_fluct_off(self.handle, _p(d), len(d), n_sigma, workers, _p(m),
                                                              _p(times)))
        return dict(sample_s=times[0], scatter_s=times[1], convolve_s=times[2], m=m)

    def __del__(self):
        try:
            self.ref.lib.wsr_plane_destroy(self.handle)
        except Exception:
            pass


def impact_charge(g, depos, impacts: int, masks, n_sigma: float = 3.0):
    """CPU restatement (numpy; test infrastructure) of fluctuation-off sampling
    at impact resolution — the extension ws_plane_create_impacts implements,
    which the reference does not have. It follows
    sample_patch (rasterize.cpp:66-120) with map_depo_to_grid's footprint and
    clip (core.cpp:25-41): the wire axis of the footprint is split into
    `impacts` sub-bins per wire, each the Gaussian's integral
    (gauss_bin_integrals, rasterize.cpp:44-64, at spacing pitch / impacts;
    sigma <= 0: the containing sub-bin), the patch normalised over all
    sub-bins x ticks. Returns one float64 charge grid per class mask
    (S_c[w, t] = q sum_{i in c} p[w, i, t]) and the clipped charge."""
    from math import ceil, erf, floor, sqrt
    W, T = padded(g)
    out = [np.zeros((W, T)) for _ in masks]
    clipped = 0

    def integrals(center, sigma, lo, spacing, n):
        v = np.zeros(n)
        if sigma <= 0.0:
            v[min(max(int(floor((center - lo) / spacing)), 0), n - 1)] = 1.0
            return v
        inv = 1.0 / (sqrt(2.0) * sigma)
        e = [erf((lo + k * spacing - center) * inv) for k in range(n + 1)]
        return 0.5 * (np.array(e[1:]) - np.array(e[:-1]))

    for d in np.asarray(depos):
        cw = int(g.pad_wires) + floor((d["x"] - g.origin_x) / g.pitch)
        ct = int(g.pad_ticks) + floor((d["t"] - g.origin_t) / g.tick)
        hw = 0 if d["sigma_x"] <= 0 else ceil(n_sigma * d["sigma_x"] / g.pitch)
        ht = 0 if d["sigma_t"] <= 0 else ceil(n_sigma * d["sigma_t"] / g.tick)
        w0, w1 = max(cw - hw, 0), min(cw + hw, W - 1)
        t0, t1 = max(ct - ht, 0), min(ct + ht, T - 1)
        if w0 > w1 or t0 > t1:
            clipped += int(d["q"])
            continue
        nw, nt = w1 - w0 + 1, t1 - t0 + 1
        wlo = g.origin_x + (w0 - int(g.pad_wires)) * g.pitch
        tlo = g.origin_t + (t0 - int(g.pad_ticks)) * g.tick
        sub = integrals(d["x"], d["sigma_x"], wlo, g.pitch / impacts, nw * impacts).reshape(nw, impacts)
        tv = integrals(d["t"], d["sigma_t"], tlo, g.tick, nt)
        total = sub.sum() * tv.sum()
        if not total > 0.0:
            clipped += int(d["q"])
            continue
        for c, m in enumerate(masks):
            wv = sub[:, [i for i in range(impacts) if (m >> i) & 1]].sum(axis=1)
            out[c][w0:w1 + 1, t0:t1 + 1] += float(d["q"]) * np.outer(wv, tv) / total
    return out, clipped
