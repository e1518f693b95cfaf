"""The GPU real-FFT backend against the reference's transform contract
(test_poisson.py:273-283: irfftn(rfftn(x)) within 4 ulp of max|x|, dtype
preserved) and against numpy's pocketfft on the same inputs, on both the
hand-written engine and the cuFFT path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2604_18536_b200 import transforms

    return transforms


def test_round_trip_contract(T):
    rng = np.random.default_rng(12)
    for shape in ((16, 16), (8, 8, 8), (7, 5)):
        for dt in (np.float64, np.float32):
            x = rng.standard_normal(shape).astype(dt)
            y = T.irfftn(T.rfftn(x), s=shape)
            bound = 4 * np.spacing(np.max(np.abs(x)))
            assert y.dtype == dt
            assert np.max(np.abs(y - x)) <= bound


@pytest.mark.parametrize("shape,own", [((16,), True), ((840, 32), True), ((64, 48, 40), True), ((12, 840, 16), True),
                                       ((1024, 6), True), ((7, 5), False), ((22, 26), False), ((9, 10, 11), False)])
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_matches_numpy(T, shape, own, dt):
    import torch

    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape).astype(dt)
    assert T.uses_own_engine(shape, dt) == own
    got = T.rfftn(torch.from_numpy(x).cuda())
    ref = np.fft.rfftn(x.astype(np.float64))
    assert got.dtype == (torch.complex128 if dt == np.float64 else torch.complex64)
    g = got.cpu().numpy()
    t = 1e-13 if dt == np.float64 else 2e-6
    assert np.max(np.abs(g - ref)) <= t * np.max(np.abs(ref))
    back = T.irfftn(got, s=shape)
    assert back.dtype == torch.from_numpy(x).dtype and tuple(back.shape) == shape
    assert np.max(np.abs(back.cpu().numpy() - x)) <= (1e-14 if dt == np.float64 else 2e-6) * np.max(np.abs(x))
    # irfftn leaves its input untouched
    assert np.array_equal(got.cpu().numpy(), g)
    # scipy-style default s (last extent 2 (m - 1)) for even shapes
    if shape[-1] % 2 == 0:
        assert np.array_equal(T.irfftn(got).cpu().numpy(), back.cpu().numpy())


def test_rejects_partial_axes_and_padding(T):
    x = np.zeros((8, 8))
    with pytest.raises(ValueError):
        T.rfftn(x, axes=(1,))
    with pytest.raises(ValueError):
        T.rfftn(x, s=(16, 8))
    with pytest.raises(ValueError):
        T.irfftn(np.zeros((8, 5), np.complex128), s=(8, 16))
