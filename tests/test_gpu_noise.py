"""GPU add_noise (white) + digitize vs the CPU oracle (wsoracle.c's
restatement of spectral.cpp:177-196 and 228-238, itself checked against the
unmodified reference in test_oracle.py). The oracle adds its noise to the
same float32 frame the GPU starts from, so the comparison isolates the noise
stream and the ADC rule."""
import numpy as np
import pytest

from paper_2104_08265_b200 import GridSpec, Plane, ResponseParams, SimConfig, WsError
from paper_2104_08265_b200.workloads import line_tracks

from .helpers import oracle_grid, relL2_per_channel

pytestmark = pytest.mark.gpu

GRID = GridSpec(n_wires=60, n_ticks=601, pad_wires=10, pad_ticks=100, pitch=5.0, tick=0.5)  # odd padded ticks


@pytest.fixture(scope="module")
def frame(ctx):
    resp = ResponseParams(plane_kind="induction", wire_weights=(0.1, 1.0, 0.1))
    plane = Plane(ctx, GRID, resp)
    m = plane.simulate(line_tracks(300, GRID, seed=2), SimConfig(grid=GRID, response=resp, fluctuate=False)).frame
    return plane, m


@pytest.mark.parametrize("rng,mode", [("substream", 0), ("philox", 1)])
def test_white_noise_and_adc(frame, oracle, rng, mode):
    import torch
    plane, m = frame
    fd = torch.from_numpy(m.copy()).cuda()
    adc = torch.empty(m.shape, dtype=torch.int32, device="cuda")
    plane.noise_digitize_device(fd, sigma=3.0, seed=77, rng=rng, adc_dev=adc, scale=0.5, offset=2048.0, bits=12)
    plane.ctx.synchronize()
    ref = oracle.add_white_noise(oracle_grid(GRID), m.astype(np.float64), 3.0, 77, rng_mode=mode)
    got = fd.cpu().numpy()
    # float32 storage of the noisy sample; the normals agree to libm ulps
    assert np.max(np.abs(got - ref)) <= 1e-6 * (np.max(np.abs(ref)) + 1.0)
    assert relL2_per_channel(got, ref) < 1e-6
    adc_ref = oracle.digitize(ref, 0.5, 2048.0, 12)
    diff = np.abs(adc.cpu().numpy().astype(np.int64) - adc_ref)
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-5  # +-1 only at an exact .5 tie moved by an ulp


def test_digitize_only_exact(frame, oracle):
    import torch
    plane, m = frame
    fd = torch.from_numpy(m.copy()).cuda()
    adc = torch.empty(m.shape, dtype=torch.int32, device="cuda")
    plane.noise_digitize_device(fd, sigma=0.0, adc_dev=adc, scale=3.0, offset=100.0, bits=10)  # clamps both ends
    plane.ctx.synchronize()
    np.testing.assert_array_equal(adc.cpu().numpy(), oracle.digitize(m.astype(np.float64), 3.0, 100.0, 10))
    np.testing.assert_array_equal(fd.cpu().numpy(), m)  # sigma 0: the frame is untouched


def test_noise_errors(frame):
    import torch
    plane, m = frame
    fd = torch.from_numpy(m.copy()).cuda()
    adc = torch.empty(m.shape, dtype=torch.int32, device="cuda")
    with pytest.raises(WsError) as e:
        plane.noise_digitize_device(fd, sigma=-1.0)
    assert e.value.code == 1 and "sigma" in str(e.value)
    with pytest.raises(WsError) as e:
        plane.noise_digitize_device(fd, adc_dev=adc, bits=17)
    assert e.value.code == 1 and "bits" in str(e.value)


SPEC_GRID = GridSpec(n_wires=60, n_ticks=600, pad_wires=10, pad_ticks=100, pitch=5.0, tick=0.5)  # 800 = 2^5 5^2 ticks
SALT = 0x737065636e6f6973  # kSpectrumNoiseSalt, spectral.cpp:22


def _spectrum(n):
    k = np.arange(n)
    f = np.minimum(k, n - k)
    return 3.0 / (1.0 + f / 40.0)


@pytest.fixture(scope="module")
def spec_frame(ctx):
    resp = ResponseParams(plane_kind="collection")
    plane = Plane(ctx, SPEC_GRID, resp)
    m = plane.simulate(line_tracks(200, SPEC_GRID, seed=4),
                       SimConfig(grid=SPEC_GRID, response=resp, fluctuate=False)).frame
    return plane, m


def test_spectrum_noise_vs_reference(spec_frame, ref):
    """Spectrum mode with the reference's own per-wire stream against the
    unmodified reference's add_noise + digitize (oracle/_ref)."""
    import torch
    plane, m = spec_frame
    amp = _spectrum(m.shape[1])
    fd = torch.from_numpy(m.copy()).cuda()
    adc = torch.empty(m.shape, dtype=torch.int32, device="cuda")
    plane.noise_digitize_device(fd, seed=31, rng="substream", adc_dev=adc, scale=2.0, offset=1000.0, bits=12,
                                spectrum=amp)
    plane.ctx.synchronize()
    noisy, adc_ref = ref.noise_digitize(oracle_grid(SPEC_GRID), m.astype(np.float64), noise_mode=2, spectrum=amp,
                                        seed=31, adc=(2.0, 1000.0, 12))
    got = fd.cpu().numpy()
    # per channel: signal rows are dominated by the frame, the padding rows
    # hold the noise waveform alone (float32 storage of frame + noise)
    assert relL2_per_channel(got, noisy) < 1e-5
    assert np.max(np.abs(got - noisy)) <= 1e-5 * np.max(np.abs(noisy))
    diff = np.abs(adc.cpu().numpy().astype(np.int64) - adc_ref)
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3


def test_spectrum_noise_philox(spec_frame, ref):
    """Philox mode: the same synthesis from the shared counter-based stream
    (uniforms from the reference-side PhiloxSource), numpy's inverse FFT."""
    import torch
    plane, m = spec_frame
    n = m.shape[1]
    amp = _spectrum(n)
    fd = torch.from_numpy(m.copy()).cuda()
    plane.noise_digitize_device(fd, seed=5, rng="philox", spectrum=amp)
    plane.ctx.synchronize()
    want = np.empty(m.shape)
    half = n // 2
    for w in range(m.shape[0]):
        u = ref.draws(1, 0, 5 ^ SALT, w, half + 1)
        x = np.zeros(n, dtype=np.complex128)
        x[0] = amp[0] * np.cos(2 * np.pi * u[0])
        x[1:half] = amp[1:half] * np.exp(2j * np.pi * u[1:half])
        x[half] = amp[half] * np.cos(2 * np.pi * u[half])
        x[half + 1:] = np.conj(x[1:half][::-1])
        want[w] = np.fft.ifft(x).real
    assert relL2_per_channel(fd.cpu().numpy(), m.astype(np.float64) + want) < 1e-5


def test_spectrum_noise_errors(spec_frame, ctx):
    import torch
    plane, m = spec_frame
    fd = torch.from_numpy(m.copy()).cuda()
    with pytest.raises(WsError) as e:
        plane.noise_digitize_device(fd, spectrum=np.ones(7))
    assert e.value.code == 1 and "amplitude_spectrum" in str(e.value)
    folded = Plane(ctx, GridSpec(n_wires=20, n_ticks=6000, pad_wires=5, pad_ticks=100), ResponseParams())  # 6200 ticks
    fd2 = torch.zeros((30, 6200), dtype=torch.float32, device="cuda")
    with pytest.raises(WsError) as e:
        folded.noise_digitize_device(fd2, spectrum=np.ones(6200))
    assert e.value.code == 1 and "7-smooth" in str(e.value)
