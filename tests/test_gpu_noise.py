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
