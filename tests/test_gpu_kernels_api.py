"""The drop-in kernels.hpp entry points that run on the device
(include/swe/kernels.hpp -> swe_dev_point_eval kinds 5-9, swe_dev_stable_dt,
swe_dev_mass) against the reference itself (oracle/_ref, the unmodified
kernels.hpp compiled in place): bit-identical on random wet / dry / straddling
inputs (reference kernels.hpp:21-216)."""
import numpy as np
import pytest

from conftest import bit_equal
from paper_1807_00672_b200 import api
from test_gpu_parity import rng_pairs

pytestmark = pytest.mark.gpu


def test_physical_flux_normal(refo):
    l, _, nrm, _ = rng_pairs(50_000, 21)
    assert bit_equal(api.point_eval(5, l, None, None, nrm), refo.point(5, l, None, None, nrm))


def test_wave_speed_estimates(refo):
    """Both dry-front branches, the two-rarefaction branch and the
    |den| < 1e-14 contact guard (kernels.hpp:38-66)."""
    l, r, _, _ = rng_pairs(50_000, 22)
    ul = np.stack([l[:, 0], np.random.default_rng(1).uniform(-3, 3, len(l)), l[:, 2]], 1)
    ur = np.stack([r[:, 0], np.random.default_rng(2).uniform(-3, 3, len(r)), r[:, 2]], 1)
    ur[:500] = ul[:500] * [1, -1, 1]  # symmetric pairs: den == 0
    ur[500:1000, 0] = ul[500:1000, 0]
    dev = api.point_eval(6, ul, ur)
    ref = refo.point(6, ul, ur)
    assert bit_equal(dev, ref)


def test_hydrostatic_reconstruct(refo):
    l, r, nrm, z = rng_pairs(50_000, 23)
    z[:2000, 1] = z[:2000, 0]  # flat edges keep both states
    assert bit_equal(api.point_eval(7, l, r, z, nrm), refo.point(7, l, r, z, nrm))


def test_cell_signal_speed(refo):
    l, _, _, _ = rng_pairs(50_000, 24)
    assert bit_equal(api.point_eval(8, l), refo.point(8, l))


def test_clamp_dry(refo):
    rng = np.random.default_rng(25)
    h = np.concatenate([rng.uniform(-2e-14, 2e-6, 20_000), [-1e-3, -0.0, 0.0, 1e-6, -1e-14, -1e-300]])
    u = np.stack([h, rng.uniform(-1, 1, len(h)), rng.uniform(-1, 1, len(h))], 1)
    dev = api.point_eval(9, u)
    assert bit_equal(dev, refo.point(9, u))
    assert dev[:, 4].sum() > 0  # the throwing branch is exercised


def test_stable_dt(refo):
    rng = np.random.default_rng(26)
    n = 200_000
    h = rng.uniform(0, 3, n)
    h[rng.random(n) < 0.3] = 0.0
    qx, qy, r = h * rng.uniform(-2, 2, n), h * rng.uniform(-2, 2, n), rng.uniform(0.1, 2, n)
    assert api.stable_dt(h, qx, qy, r) == refo.stable_dt(h, qx, qy, r)[0]
    z = np.zeros(4)
    assert api.stable_dt(z, z, z, np.ones(4)) == 1.0  # all dry -> dt_max
    qx[[17, 3, 99]] = np.nan
    h[[17, 3, 99]] = 1.0
    _, bad = refo.stable_dt(h, qx, qy, r)
    assert bad == 3
    with pytest.raises(api.NumericError, match=r"non-finite velocity in cell 3$"):
        api.stable_dt(h, qx, qy, r)


def test_mass_is_stateless_and_close_to_serial():
    rng = np.random.default_rng(27)
    h, a = rng.uniform(0, 2, 1_000_003), rng.uniform(0.5, 1.5, 1_000_003)
    ref = float(np.sum(h * a, dtype=np.float64))
    m = api.mass(h, a)
    assert m == api.mass(h, a)  # fixed order
    assert abs(m - ref) <= 1e-13 * ref
