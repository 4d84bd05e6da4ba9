"""Device GRF sampler (lt_sample_field_grid, the structured-grid replacement of
sample_field_on_mesh, fields.cpp:84-123): parity with the NumPy circulant-embedding restatement
(paper_1409_2556_b200/inputs.py) on shared noise, and the statistics of the Philox path."""
import numpy as np
import pytest

from paper_1409_2556_b200 import inputs
from paper_1409_2556_b200 import laptomo as L

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return L.Context(0)


@pytest.mark.parametrize("shape,corr", [((24, 20), (0.2, 0.1)), ((16, 12, 10), (0.2, 0.2, 0.05)),
                                        ((7, 9, 5), (0.3, 0.1, 0.2))])
def test_sample_field_matches_numpy_on_shared_noise(ctx, shape, corr):
    h = 1.0 / shape[0]
    ext = [2 * n for n in shape]
    rng = np.random.default_rng(11)
    xi = rng.standard_normal(ext) + 1j * rng.standard_normal(ext)  # indexed (x, y[, z])
    ref = inputs.grf_exponential(shape, h, 1.7, corr, -9.0, 0, noise=xi).ravel()
    got = L.sample_field_grid(ctx, shape, h, 1.7, corr, -9.0, noise=np.transpose(xi))  # x fastest
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref - (-9.0)))


def test_sample_field_philox_statistics(ctx):
    shape, h, var, ell = (16, 16, 16), 1.0 / 16, 1.0, 0.2
    a = L.sample_field_grid(ctx, shape, h, var, (ell,) * 3, 2.0, seed=5)
    b = L.sample_field_grid(ctx, shape, h, var, (ell,) * 3, 2.0, seed=5)
    c = L.sample_field_grid(ctx, shape, h, var, (ell,) * 3, 2.0, seed=6)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    draws = np.stack([L.sample_field_grid(ctx, shape, h, var, (ell,) * 3, 2.0, seed=s) for s in range(64)])
    dev = draws - 2.0
    # pointwise variance over the draws, averaged over the cells: var
    assert abs(np.mean(dev * dev) / var - 1.0) < 0.1
    # correlation of x-neighbours: exp(-h / l)
    f = dev.reshape(64, 16, 16, 16)
    rho = np.mean(f[..., 1:] * f[..., :-1]) / np.mean(dev * dev)
    assert abs(rho - np.exp(-h / ell)) < 0.05


def test_sample_field_rejects_bad_arguments(ctx):
    with pytest.raises(ValueError):
        L.sample_field_grid(ctx, (8, 8), 0.1, 1.0, (0.2,), 0.0)
    with pytest.raises(ValueError):
        L.sample_field_grid(ctx, (8, 8), -0.1, 1.0, (0.2, 0.2), 0.0)
